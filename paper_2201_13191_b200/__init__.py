"""B200-native Monte Carlo scatter / primary forward projector.

Drop-in for the projector path of the reference xscat library
(include/xscat/transport.hpp:69-116, postprocess.hpp:13-41): hand-written
sm_100a CUDA kernels behind the C ABI of include/xscat_gpu.h
(lib/libxscatgpu.so), with this package as the host-side mirror of the
reference API.  See DESIGN.md.
"""
from . import configs, inputs, synthetic  # noqa: F401
from .inputs import (DetectorResponse, Material, ScanGeometry, SimConfig, Spectrum,  # noqa: F401
                     Table1D, VoxelPhantom, XscatError, XscatInvalidArgument,
                     XscatOutOfRange, detector_response, kramers_spectrum, load_detector_response,
                     load_material, load_spectrum, make_circular_geometry, make_empty_phantom,
                     material, monochromatic_spectrum, spectrum)
from .projector import (BOTH, HANN, PRIMARY, RAMLAK, SCATTER, Context, Group, ProjectionStack, Projector,  # noqa: F401
                        ScanResult, SgFilterSpec, SimResult, WeightLedger, apportion_photons,
                        correct_projections, correction_tail, default_sg_spec, default_voxel_size,
                        device_count, fbp_reconstruct,
                        downsample_average, finalize_host, intensity_to_attenuation,
                        history_count, interpolate_angles, point_detector_score, run_scan,
                        sg_kernel, sg_smooth, simulate_primary, simulate_scatter,
                        simulate_scatter_stats, upsample_image, ClassSpec, SegmentationResult,
                        otsu_thresholds, segment_volume, to_density_phantom, segment_to_scene,
                        CorrectionConfig, CorrectionResult, IterationReport, run_iterative_correction)

__version__ = "0.1.0"
