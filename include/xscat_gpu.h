/*
 * xscat_gpu.h — C ABI of the B200-native Monte Carlo scatter / primary
 * forward projector (drop-in for the reference xscat projector path).
 *
 * The reference (`/root/reference/proj`, "REF") has no FFI: its boundary is
 * the C++ API in include/xscat/transport.hpp:69-116 and
 * include/xscat/postprocess.hpp:13-41.  Every entry point below replaces one
 * of those functions; the citation is given per declaration.  Plain pointers
 * and sizes only; no C++ or torch types cross this boundary.
 *
 * Conventions
 *  - Every function returns an xs_status; XS_OK == 0.  Non-zero codes map
 *    one-to-one onto the exception types REF throws (see xs_status), and the
 *    message REF would have put into e.what() is available from
 *    xs_last_error(ctx) (ctx may be NULL for context-free calls: the message
 *    is then thread-local).
 *  - Host buffers are owned by the caller.  Device buffers created by the
 *    library are owned by the context.  One context = one CUDA device + one
 *    stream; a context is not thread-safe, distinct contexts are.
 *  - Images are fp64, row-major, index iv*nu + iu (REF detector_image.hpp:11-22).
 *  - Voxel arrays are x-fastest, index ix + nx*(iy + ny*iz) (REF phantom.hpp:14-37).
 */
#ifndef XSCAT_GPU_H
#define XSCAT_GPU_H

#include <math.h>
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XS_ABI_VERSION 1

/* ------------------------------------------------------------------ status */
typedef enum xs_status {
    XS_OK = 0,
    XS_E_RUNTIME = 1,          /* REF throws std::runtime_error            */
    XS_E_OUT_OF_RANGE = 2,     /* REF throws std::out_of_range             */
    XS_E_INVALID_ARGUMENT = 3, /* REF throws std::invalid_argument         */
    XS_E_DOMAIN = 4,           /* REF throws std::domain_error             */
    XS_E_CUDA = 5,             /* CUDA runtime failure (no REF counterpart) */
    XS_E_UNSUPPORTED = 6       /* input beyond the device path's limits    */
} xs_status;

/* ------------------------------------------------------------ input types */

/* One strictly-increasing 1-D table (REF table.hpp:15-95). */
typedef struct xs_table {
    int32_t n;
    const double* x;
    const double* y;
} xs_table;

/* REF material.hpp:15-32.  The F^2 dq^2 CDF (REF material.cpp:107-125) is
 * derived by the library from f_factor; callers do not supply it. */
typedef struct xs_material {
    const char* name;
    double z_eff;
    double density_ref;
    xs_table mu;          /* keV -> cm^2/g, log-log        */
    xs_table sigma_incoh; /* keV -> barn, log-log          */
    xs_table sigma_coh;   /* keV -> barn, log-log          */
    xs_table sigma_pe;    /* keV -> barn, log-log          */
    xs_table s_factor;    /* 1/A -> S, linear, clamp z_eff */
    xs_table f_factor;    /* 1/A -> F, linear, clamped     */
} xs_material;

/* REF VoxelPhantom (phantom.hpp:14-37).  materials[0] is the vacuum
 * sentinel (its tables are ignored and may be empty). */
typedef struct xs_phantom {
    int32_t dims[3];
    double voxel_size[3]; /* cm */
    double origin[3];     /* low corner, cm */
    const uint8_t* material_id;
    const float* density; /* g/cm^3 */
    int32_t n_materials;  /* including vacuum at index 0 */
    const xs_material* materials;
} xs_phantom;

/* REF ScanGeometry (scan_geometry.hpp:20-40). */
typedef struct xs_geometry {
    double sdd;
    double sod;
    int32_t nu;
    int32_t nv;
    double pixel_pitch;
    int32_t n_angles;
    const double* angles; /* radians, strictly increasing in [0, 2pi) */
} xs_geometry;

/* REF Spectrum (spectrum.hpp:14-26). */
typedef struct xs_spectrum {
    int32_t n_bins;
    const double* energy_kev;
    const double* weight;
} xs_spectrum;

/* REF DetectorResponse (detector_response.hpp:11-24). */
typedef struct xs_response {
    xs_table dqe;
    xs_table deposit;
} xs_response;

/* REF SimConfig (transport.hpp:22-31); same defaults via xs_sim_config_default. */
typedef struct xs_sim_config {
    uint64_t photons_total;
    int32_t splitting;
    double roulette_survival;
    double roulette_wmin_rel;
    int32_t step_voxels;
    int32_t max_interactions;
    uint64_t seed;
    int32_t track_variance;
} xs_sim_config;

/* REF WeightLedger (transport.hpp:38-56). */
typedef struct xs_ledger {
    double initial;
    double escaped;
    double absorbed;
    double culled;
    double roulette_killed;
    double roulette_boost;
} xs_ledger;

/* REF SimResult (transport.hpp:58-64).  image (nu*nv) is required;
 * variance (nu*nv) is written only when track_variance and non-NULL. */
typedef struct xs_scatter_result {
    double* image;
    double* variance;
    xs_ledger ledger;
    uint64_t histories;
    double total;
    double total_std_error;
} xs_scatter_result;

/* Per-launch device counters (the roofline numerator). */
typedef struct xs_launch_stats {
    uint64_t free_path_steps;  /* voxel visits of the free-path walks          */
    uint64_t scoring_steps;    /* voxel visits (or midpoint samples) of scoring rays */
    uint64_t histories;        /* histories processed by the launch          */
    uint64_t scoring_rays;     /* next-event pseudo-particles traced          */
    uint64_t interactions;     /* Compton + Rayleigh + photoelectric events   */
    double kernel_ms;          /* transport kernel time, CUDA events          */
    int32_t voxel_format;      /* 0 = 4-bit palette, 1 = 8-bit palette, 2 = raw id+density */
    int32_t palette_size;
    uint64_t upload_bytes;     /* encoded voxel bytes of the last phantom upload (H2D) */
    uint64_t walk_iterations;  /* walker loop iterations (< steps when macro cells are skipped) */
    uint64_t walk_lane_slots;  /* 32 x warp-level walker iterations (lane occupancy denominator) */
    uint32_t blocks_per_sm;    /* resident transport blocks per SM */
    uint32_t smem_per_block;   /* dynamic shared memory per transport block (bytes) */
    uint32_t slots_per_warp;   /* live histories per warp (megakernel) */
    uint32_t engine;           /* 0: persistent megakernel, 1: wavefront pipeline */
    uint32_t waves;            /* wavefront: pipeline waves run */
    uint32_t live_histories;   /* histories in flight at once */
    uint64_t uniform_iterations; /* walker iterations that crossed a uniform cell / brick */
    float walk_ms;             /* device time of the walk kernel(s) (the whole kernel for the megakernel) */
    uint32_t launches;         /* kernels launched by the scatter call */
    uint32_t block_walk;       /* 1: the walk crossed uniform blocks (walk_mode, per-phantom probe) */
    /* environment XSCAT_KTIME=1 (wavefront engine): summed device time of the
     * other kernels of every wave, CUDA events on the pipeline streams */
    float setup_ms, score_ms, event_ms, admit_ms;
} xs_launch_stats;

typedef struct xs_context xs_context;

/* ------------------------------------------------- deterministic accumulator
 *
 * Scatter tallies are accumulated as exact integers so the result is
 * bit-identical for any thread schedule and any number of GPUs.  A
 * non-negative real x is stored relative to a power-of-two unit U as three
 * 32-bit limbs of the 96-bit fixed-point number x/U * 2^64:
 *   limb2 = floor(x/U), limb1 = next 32 bits, limb0 = last 32 bits (rounded).
 * Each limb is added into its own uint64 slot, so a slot absorbs 2^32 adds
 * without overflow and limb sums from several GPUs can be added by a plain
 * integer sum-reduce (NCCL ncclUint64/ncclInt64 ncclSum).
 *
 * Layout of one accumulator buffer (uint64 words), see xs_accum_layout():
 *   image    : 4 words per pixel  {limb0, limb1, limb2, 0}   unit U_img
 *   variance : 4 words per pixel  (track_variance only)      unit U_img^2
 *   bins     : 8 words per bin    {T limbs[3], T^2 limbs[3], 0, 0}
 *   ledger   : 6 x 4 words        initial, escaped, absorbed, culled,
 *                                 roulette_killed, roulette_boost; unit U_w
 *   diag     : 8 words            launch counters (xs_launch_stats order)
 */
typedef struct xs_accum_layout {
    uint64_t n_pixels;
    uint64_t off_image;
    uint64_t off_variance; /* == off_bins when variance is not tracked */
    uint64_t off_bins;
    uint64_t off_ledger;
    uint64_t off_diag;
    uint64_t words;
} xs_accum_layout;

static inline xs_accum_layout xs_accum_layout_make(int32_t nu, int32_t nv, int32_t n_bins,
                                                   int32_t track_variance)
{
    xs_accum_layout l;
    l.n_pixels = (uint64_t)nu * (uint64_t)nv;
    l.off_image = 0;
    l.off_variance = 4 * l.n_pixels;
    l.off_bins = l.off_variance + (track_variance ? 4 * l.n_pixels : 0);
    l.off_ledger = l.off_bins + 8 * (uint64_t)n_bins;
    l.off_diag = l.off_ledger + 24;
    l.words = l.off_diag + 8;
    return l;
}

/* Power-of-two units of the fixed-point tallies; functions of the inputs
 * only (never of the GPU count), so every split of the history range
 * produces limbs in the same units.
 *   U_img = 2^floor(log2(sum_b w_b / sdd^2))   (flat-field scale; response <= 1)
 *   U_w   = 2^ceil(log2(max_b(w_b / M_b) * A_det / sdd^2))   (bound on w0)   */
typedef struct xs_accum_units {
    int32_t log2_img;
    int32_t log2_w;
} xs_accum_units;

static inline int32_t xs__floor_log2(double v)
{
    int e = 0;
    if (!(v > 0.0) || !isfinite(v))
        return 0;
    (void)frexp(v, &e); /* v = m 2^e, m in [0.5, 1) */
    return (int32_t)(e - 1);
}

static inline int32_t xs__ceil_log2(double v)
{
    int e = 0;
    double m;
    if (!(v > 0.0) || !isfinite(v))
        return 0;
    m = frexp(v, &e);
    return (int32_t)(m == 0.5 ? e - 1 : e);
}

static inline xs_accum_units xs_accum_units_make(const xs_geometry* g, const xs_spectrum* s,
                                                 const uint64_t* photons_per_bin)
{
    xs_accum_units u;
    double wsum = 0.0, wmax = 0.0;
    const double sdd2 = g->sdd * g->sdd;
    const double area = (double)g->nu * (double)g->nv * g->pixel_pitch * g->pixel_pitch;
    int32_t b;
    for (b = 0; b < s->n_bins; ++b) {
        wsum += s->weight[b];
        if (photons_per_bin[b] > 0) {
            const double r = s->weight[b] / (double)photons_per_bin[b];
            if (r > wmax)
                wmax = r;
        }
    }
    u.log2_img = xs__floor_log2(wsum / sdd2);
    u.log2_w = xs__ceil_log2(wmax * area / sdd2);
    return u;
}

/* Splits q = x/U (0 <= q < 2^32) into the three limbs; every step is exact
 * in IEEE binary64 except the final round-half-even, so host and device
 * produce identical limbs.  Returns 0 on success, 1 if q is out of range. */
static inline int xs_quantize(double q, uint64_t limb[3])
{
    double i2, r, r1, i1, r2;
    if (!(q >= 0.0) || !(q < 4294967296.0))
        return 1;
    i2 = floor(q);
    r = q - i2;
    r1 = r * 4294967296.0;
    i1 = floor(r1);
    r2 = (r1 - i1) * 4294967296.0;
    limb[2] = (uint64_t)i2;
    limb[1] = (uint64_t)i1;
    limb[0] = (uint64_t)nearbyint(r2);
    return 0;
}

/* Exact limb sum back to a double in units of U (deterministic rounding). */
static inline double xs_dequantize(const uint64_t* s, int32_t log2_unit)
{
    /* S = s2*2^64 + s1*2^32 + s0 as a 128-bit integer (hi, lo) */
    uint64_t lo = s[0];
    uint64_t hi = s[2];
    uint64_t t = s[1] << 32;
    uint64_t c = s[1] >> 32;
    uint64_t lo2 = lo + t;
    hi += c + (lo2 < lo ? 1u : 0u);
    lo = lo2;
    return ldexp((double)hi * 18446744073709551616.0 + (double)lo, log2_unit - 64);
}

/* ------------------------------------------------------------ host helpers */

const char* xs_version(void);
int xs_abi_version(void);

/* Thread-local message of the last failing call (context-free calls). */
const char* xs_last_error(const xs_context* ctx);

/* REF SimConfig{} defaults (transport.hpp:22-31). */
void xs_sim_config_default(xs_sim_config* cfg);

/* REF validate_sim_config (transport.cpp:26-40). */
int xs_validate_sim_config(const xs_sim_config* cfg);

/* REF apportion_photons (transport.cpp:42-64); counts has n_bins entries. */
int xs_apportion_photons(const xs_spectrum* spec, uint64_t photons_total, uint64_t* counts);

/* REF point_detector_score (transport.cpp:66-71). */
double xs_point_detector_score(double response_factor, double p_dir, double weight,
                               double n_pixels, double d2, double tau);

/* Finalize a (possibly reduced) accumulator on the host, no GPU needed:
 * REF simulate_scatter_stats ordered reduction + SE + variance
 * (transport.cpp:289-322).  hist_begin/hist_end is the global history range
 * the accumulator covers (the whole range after a reduce). */
int xs_scatter_finalize_host(const xs_geometry* g, const xs_spectrum* spec,
                             const xs_sim_config* cfg, const uint64_t* accum,
                             uint64_t hist_begin, uint64_t hist_end, xs_scatter_result* out);

/* Total number of histories (sum of apportioned photons) of a run. */
int xs_history_count(const xs_spectrum* spec, uint64_t photons_total, uint64_t* n_histories);

/* Savitzky-Golay helpers (REF postprocess.cpp:11-102). */
int xs_validate_sg_spec(int32_t window, int32_t polyorder);
int xs_default_sg_spec(int32_t nu, int32_t nv, int32_t* window, int32_t* polyorder);
int xs_sg_kernel(int32_t left, int32_t right, int32_t polyorder, double* out /* left+right+1 */);

/* --------------------------------------------------------------- context */

int xs_device_count(int32_t* n);
int xs_ctx_create(int32_t device, xs_context** out);
void xs_ctx_destroy(xs_context* ctx);
/* Use an external CUDA stream (cudaStream_t as void*); NULL restores the
 * context's own stream. */
int xs_ctx_set_stream(xs_context* ctx, void* cuda_stream);
int xs_ctx_synchronize(xs_context* ctx);

/* Tuning / mode knobs (no REF counterpart):
 *   "exact_walk"  1: voxel-by-voxel Siddon everywhere (strict REF replay);
 *                 0 (default): cross uniform 8^3 macro cells in one step, which
 *                 changes the optical depths only at fp64 rounding level
 *   "smem_kb"     shared memory per transport block (8..227, default 48:
 *                 four blocks per SM keep 60 KB of L1); bounds the live
 *                 histories per warp
 *   "max_slots"   live histories per warp (1..64)
 *   "grab"        histories a warp reserves from the pool at a time
 *   "engine"      1 (default): wavefront pipeline (set-up / walk / event
 *                 kernels over global queues); 0: persistent megakernel.
 *                 Both give bit-identical results.  step_voxels > 1
 *                 (REF's march mode) always runs the megakernel
 *   "wave_slots"  histories in flight in the wavefront engine (2^24)
 *   "wave_pipes"  concurrent wavefront pipelines on their own streams (2)
 *   "compact_palette" 1: 4-bit voxel palette for <= 8 (material, density)
 *                 pairs (half the bytes); 0 (default): 8-bit palette, which
 *                 leaves room for more uniform-block levels.  Applies to the
 *                 next xs_upload_phantom
 *   "walk_mode"   0: voxel-by-voxel walk; 1: cross uniform blocks in one step;
 *                 2 (default): chosen per phantom at upload by a ray probe
 *                 (voxel-walk phantoms of <= 16 pairs are stored as 4-bit codes)
 *   "upload_path" 1 (default): xs_upload_phantom stages the host arrays
 *                 through pinned memory and validates / encodes on the device;
 *                 0: validates / encodes on the host.  Same grid either way  */
int xs_ctx_set_option(xs_context* ctx, const char* key, int64_t value);

/* Scene upload: REF passes the phantom and response by const& to every
 * projector call; here they are uploaded once and reused until replaced.
 * xs_upload_phantom validates like REF validate_phantom (phantom.cpp:33-56)
 * and re-encodes the grid into the device voxel format. */
int xs_upload_phantom(xs_context* ctx, const xs_phantom* ph);
int xs_upload_response(xs_context* ctx, const xs_response* resp);

/* ---------------------------------------------------------- the projector */

/* REF simulate_scatter_stats (transport.hpp:89-91, transport.cpp:246-324):
 * whole history range on this device, host outputs. */
int xs_simulate_scatter_stats(xs_context* ctx, const xs_geometry* g, int32_t angle_idx,
                              const xs_spectrum* spec, const xs_sim_config* cfg,
                              xs_scatter_result* out);

/* REF simulate_primary (transport.hpp:100-102, transport.cpp:333-377):
 * image_host has nu*nv doubles. */
int xs_simulate_primary(xs_context* ctx, const xs_geometry* g, int32_t angle_idx,
                        const xs_spectrum* spec, const xs_sim_config* cfg, double* image_host);

/* REF run_scan (transport.hpp:112-116, transport.cpp:379-422).  what: 0 =
 * primary, 1 = scatter, 2 = both (ScanQuantity order).  primary_out /
 * scatter_out hold n_subset*nu*nv doubles (angle-major) or NULL when not
 * requested; seconds_per_angle (n_subset) may be NULL. */
int xs_run_scan(xs_context* ctx, const xs_geometry* g, const xs_spectrum* spec,
                const xs_sim_config* cfg, const int32_t* angle_subset, int32_t n_subset,
                int32_t what, double* primary_out, double* scatter_out,
                double* seconds_per_angle);

/* Device-level split of simulate_scatter_stats for photon-batch sharding
 * across GPUs: accumulate histories [hist_begin, hist_end) of the global
 * bin-major history order into the device buffer d_accum (layout above;
 * the caller zeroes it once, calls may add into the same buffer).  After a
 * sum-reduce of the buffers of all ranks, xs_scatter_finalize_device (or
 * xs_scatter_finalize_host on a D2H copy) produces the SimResult. */
int xs_scatter_accumulate_device(xs_context* ctx, const xs_geometry* g, int32_t angle_idx,
                                 const xs_spectrum* spec, const xs_sim_config* cfg,
                                 uint64_t hist_begin, uint64_t hist_end, uint64_t* d_accum);
int xs_scatter_finalize_device(xs_context* ctx, const xs_geometry* g, const xs_spectrum* spec,
                               const xs_sim_config* cfg, const uint64_t* d_accum,
                               uint64_t hist_begin, uint64_t hist_end, xs_scatter_result* out,
                               double* d_image /* optional device copy, nu*nv */);

/* Deterministic primary into a device buffer (nu*nv doubles). */
int xs_primary_device(xs_context* ctx, const xs_geometry* g, int32_t angle_idx,
                      const xs_spectrum* spec, const xs_sim_config* cfg, double* d_image);

/* Replicates ctx src's uploaded scene (encoded voxel grid, materials,
 * detector response) into ctx dst, device to device (NVLink peer copy when
 * the devices differ), without re-validating or re-encoding.  Used to give
 * every GPU of a group the phantom that was uploaded (or segmented) on one. */
int xs_ctx_copy_scene(xs_context* dst, const xs_context* src);

/* Counters of the last scatter launch. */
int xs_last_launch_stats(const xs_context* ctx, xs_launch_stats* out);

/* -------------------------------------------------------- post-processing
 * REF postprocess.hpp:17-41, batched over n_images images of one grid.
 * device_ptrs = 0: in/out are host pointers; 1: device pointers. */

/* REF sg_smooth (postprocess.cpp:124-145). */
int xs_sg_smooth(xs_context* ctx, const double* in, double* out, int32_t nu, int32_t nv,
                 int32_t n_images, int32_t window, int32_t polyorder, int32_t device_ptrs);

/* REF interpolate_angles (postprocess.cpp:147-196): in holds n_src images at
 * src_angles, out receives n_tgt images at tgt_angles. */
int xs_interpolate_angles(xs_context* ctx, const double* in, const double* src_angles,
                          int32_t n_src, double* out, const double* tgt_angles, int32_t n_tgt,
                          int32_t nu, int32_t nv, int32_t device_ptrs);

/* REF upsample_image (postprocess.cpp:235-252). */
int xs_upsample_image(xs_context* ctx, const double* in, int32_t nu, int32_t nv,
                      int32_t n_images, double* out, int32_t nu_out, int32_t nv_out,
                      int32_t device_ptrs);

/* REF downsample_average (postprocess.cpp:254-271). */
int xs_downsample_average(xs_context* ctx, const double* in, int32_t nu, int32_t nv,
                          int32_t n_images, double* out, int32_t nu_out, int32_t nv_out,
                          int32_t device_ptrs);

/* ------------------------------------------------ correction-loop stages
 * (the elementwise stages that follow the projector
 * in REF's iterative correction).  Stacks are n_images row-major images;
 * device_ptrs as above.  Errors carry REF's messages (runtime_error). */

/* REF intensity_to_attenuation (recon.cpp:324-348): a = ln(flat / I). */
int xs_intensity_to_attenuation(xs_context* ctx, const double* intensity, const double* flatfield,
                                int32_t nu, int32_t nv, int32_t n_images, double* out,
                                int32_t device_ptrs);

/* REF correct_projections (correction.cpp:58-86), Eq. 8:
 * c = a - ln(Ip / (Ip + max(Is, 0))); *clamped = negative-scatter pixels. */
int xs_correct_projections(xs_context* ctx, const double* a, const double* primary,
                           const double* scatter, int32_t nu, int32_t nv, int32_t n_images,
                           double* out, uint64_t* clamped, int32_t device_ptrs);

/* The loop's tail after the Monte Carlo runs (REF correction.cpp:199-246):
 * SG-smooth the n_sub scatter images (MC resolution nu x nv), interpolate
 * them to the n_full angles, up-sample scatter and primary (n_full images at
 * nu x nv) to nu_out x nv_out, floor each primary view at 1e-12 of its peak,
 * and apply Eq. 8 to `a` (n_full images at nu_out x nv_out).  The scatter
 * up-sampling is fused with the correction, so the full-resolution scatter
 * stack is never stored.  Returns the corrected stack, the mean scatter
 * fraction Is / (Ip + Is) and the clamped count. */
int xs_correction_tail(xs_context* ctx, const double* scatter_sub, const double* sub_angles,
                       int32_t n_sub, const double* primary_mc, const double* full_angles,
                       int32_t n_full, int32_t nu, int32_t nv, int32_t sg_window, int32_t sg_order,
                       const double* a, int32_t nu_out, int32_t nv_out, double* corrected,
                       double* mean_scatter_fraction, uint64_t* clamped, int32_t device_ptrs);

/* FDK reconstruction (REF fbp_reconstruct, recon.cpp:58-157; SURVEY.md §8(f)
 * rank 2): cosine weighting, row ramp filter (hann = 1: Hann window, 0:
 * Ram-Lak), distance-weighted bilinear backprojection.  `stack` holds
 * n_views images (nv x nu, row-major) at `angles` (ascending); the volume is
 * dims[0] x dims[1] x dims[2] floats (x fastest) in 1/m, centred on the
 * isocenter.  Same arithmetic and order as REF: bit-identical volume.
 * Errors as REF: empty stack, insufficient angular coverage (runtime_error). */
int xs_fbp_reconstruct(xs_context* ctx, const double* stack, const double* angles, int32_t n_views,
                       int32_t nu, int32_t nv, const xs_geometry* g, const int32_t dims[3],
                       const double voxel[3], int32_t hann, float* volume, int32_t device_ptrs);
/* REF default_voxel_size (recon.cpp:13-18). */
void xs_default_voxel_size(const xs_geometry* g, const int32_t dims[3], double out[3]);

/* ----------------------------------------------------------- segmentation
 * the loop's segmentation stage (REF recon.cpp:159-322,
 * correction.cpp:167-172) on the device.  Bit-identical to REF. */

/* REF ClassSpec (recon.hpp:32-35). */
typedef struct xs_class_spec {
    int32_t material_id; /* 0 = vacuum */
    double density;      /* g/cm^3 */
} xs_class_spec;

/* REF otsu_thresholds (recon.hpp:27-29, recon.cpp:159-240): n_classes - 1
 * ascending thresholds (host array) of a dims[0] x dims[1] x dims[2] float
 * volume (x fastest).  Errors as REF: invalid_argument for n_classes outside
 * [2,4] or histogram_bins < n_classes; runtime_error "degenerate histogram". */
int xs_otsu_thresholds(xs_context* ctx, const float* volume, const int32_t dims[3], int32_t n_classes,
                       int32_t histogram_bins, double* thresholds, int32_t device_ptrs);

/* REF segment_volume (recon.hpp:43-44, recon.cpp:242-262): labels[i] = number
 * of leading thresholds <= volume[i].  n_class_map = REF class_map.size()
 * (checked like REF).  thresholds are host doubles. */
int xs_segment_volume(xs_context* ctx, const float* volume, uint64_t n_voxels, const double* thresholds,
                      int32_t n_thresholds, int32_t n_class_map, uint8_t* labels, int32_t device_ptrs);

/* REF to_density_phantom (recon.hpp:50-53, recon.cpp:264-322): block mode of
 * the labels (ties to the higher label) and block mean of the class
 * densities onto target_dims; then REF validate_phantom against `materials`
 * (n_materials incl. vacuum; NULL skips it).  Errors: "unmapped label N". */
int xs_to_density_phantom(xs_context* ctx, const uint8_t* labels, const int32_t src_dims[3],
                          const xs_class_spec* class_map, int32_t n_classes, const int32_t target_dims[3],
                          int32_t n_materials, const xs_material* materials, uint8_t* material_id,
                          float* density, int32_t device_ptrs);

/* The loop's segmentation stage fused (REF correction.cpp:168-171): Otsu
 * with REF's default 1024 bins (or histogram_bins) -> labels -> density
 * phantom on target_dims, which becomes the context's scene (as if passed
 * to xs_upload_phantom) without leaving the device.  Thresholds out (host). */
int xs_segment_to_scene(xs_context* ctx, const float* volume, const int32_t dims[3], const double voxel_size[3],
                        int32_t n_classes, int32_t histogram_bins, const xs_class_spec* class_map,
                        const int32_t target_dims[3], int32_t n_materials, const xs_material* materials,
                        double* thresholds, int32_t device_ptrs);

/* xs_upload_phantom for a phantom whose material_id / density arrays are
 * device pointers (same validation, errors and device grid). */
int xs_upload_phantom_device(xs_context* ctx, const xs_phantom* ph);

/* xs_run_scan with device outputs: d_primary / d_scatter (either NULL) hold
 * n_subset images of nu x nv doubles in device memory. */
int xs_run_scan_device(xs_context* ctx, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                       const int32_t* angle_subset, int32_t n_subset, int32_t what, double* d_primary,
                       double* d_scatter, double* seconds_per_angle);

/* ------------------------------------------------- iterative correction */

/* REF CorrectionConfig (correction.hpp:13-24); defaults via
 * xs_correction_config_default.  class_map: n_classes entries. */
typedef struct xs_correction_config {
    int32_t n_iterations;
    int32_t simulate_every_kth_angle;
    int32_t mc_nu, mc_nv; /* 0 = full resolution */
    int32_t recon_dims[3];
    int32_t n_classes;
    const xs_class_spec* class_map;
    xs_sim_config sim;
    int32_t sg_window, sg_polyorder;
    int32_t sg_auto_window;
} xs_correction_config;
void xs_correction_config_default(xs_correction_config* cfg);

/* REF IterationReport (correction.hpp:26-39).  seconds_postprocess covers the
 * fused post-processing + Eq. 8 pass (seconds_correction is 0). */
typedef struct xs_iteration_report {
    int32_t iteration;
    int32_t pad_;
    double seconds_fbp, seconds_segmentation, seconds_mc_scatter, seconds_mc_primary;
    double seconds_postprocess, seconds_correction, seconds_total;
    double mc_seconds_per_projection, mean_scatter_fraction, ncc_to_previous;
    uint64_t negative_scatter_clamped;
} xs_iteration_report;

/* REF run_iterative_correction (correction.hpp:60-75, correction.cpp:137-266)
 * with every stage on the device.  raw_intensity: g->n_angles images of
 * nv x nu; flatfield: one image; materials: n_materials entries incl. vacuum
 * (REF's list + 1); the detector response comes from xs_upload_response.
 * Outputs (either may be NULL): the corrected volume (recon_dims floats) and
 * the corrected stack; reports: n_iterations entries.  device_ptrs applies
 * to raw_intensity, flatfield and both outputs.  Errors as REF, stage errors
 * prefixed "iteration N, stage S: ". */
int xs_run_iterative_correction(xs_context* ctx, const double* raw_intensity, const double* flatfield,
                                const xs_geometry* g, const xs_spectrum* spec, const xs_correction_config* cfg,
                                int32_t n_materials, const xs_material* materials, float* corrected_volume,
                                double* corrected_stack, xs_iteration_report* reports, int32_t device_ptrs);

/* ------------------------------------------------------------- multi-GPU
 * SURVEY.md §8(e).  A history is a pure function of (seed, angle, bin,
 * photon) (REF rng.hpp:13-17, transport.cpp:122-123) and the tallies are
 * integers, so one projection's history range is split into contiguous
 * photon batches, one per GPU (REF's chunk rule transport.cpp:274-275 with one
 * chunk per GPU), and the accumulators are summed: the image is bit-identical
 * for any GPU count.  Scans are split into contiguous angle ranges (REF
 * run_scan's angle loop transport.cpp:405-420).
 *
 * Multi-process (one process per GPU, e.g. torchrun): rank 0 calls
 * xs_comm_unique_id and sends the id to every rank by any channel; every rank
 * calls xs_ctx_comm_init on its context.  The context then owns an NCCL
 * communicator: accumulators are combined with ncclReduce(ncclUint64, ncclSum)
 * and scan images gathered with ncclSend/ncclRecv, on the context's stream.
 * Every rank calls the *_mgpu functions with identical arguments; if any rank
 * fails, all ranks fail (the failing rank with its own REF message). */
typedef struct xs_comm_id {
    char internal[128];
} xs_comm_id;
int xs_comm_unique_id(xs_comm_id* out);
int xs_ctx_comm_init(xs_context* ctx, int32_t n_ranks, int32_t rank, const xs_comm_id* id);
int xs_ctx_comm_size(const xs_context* ctx, int32_t* n_ranks, int32_t* rank);

/* REF simulate_scatter_stats (transport.cpp:246-324) over the communicator:
 * rank r runs histories [n r / N, n (r + 1) / N) of the bin-major order, the
 * accumulators are reduced onto `root`, which finalizes into *out (image and
 * variance as in xs_simulate_scatter_stats; out->image may be NULL) and, if
 * d_image is not NULL, into that device buffer.  Other ranks get
 * out->histories = their share and nothing else. */
int xs_simulate_scatter_stats_mgpu(xs_context* ctx, const xs_geometry* g, int32_t angle_idx,
                                   const xs_spectrum* spec, const xs_sim_config* cfg, int32_t root,
                                   xs_scatter_result* out, double* d_image);

/* REF run_scan (transport.cpp:379-422) over the communicator: rank r runs the
 * contiguous share [n r / N, n (r + 1) / N) of angle_subset and writes those
 * angles' images (and seconds) into its own outputs, laid out as for
 * xs_run_scan (n_subset images, angle-major; NULL outputs are skipped).  With
 * gather != 0 the root's outputs also receive every other rank's images. */
int xs_run_scan_mgpu(xs_context* ctx, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                     const int32_t* angle_subset, int32_t n_subset, int32_t what, int32_t gather, int32_t root,
                     double* primary_out, double* scatter_out, double* seconds_per_angle);

/* One process, several GPUs: a group of contexts, one per listed device (a
 * device may repeat; its contexts then share it).  Group calls run the members
 * concurrently, one host thread each.  The photon batches of one projection
 * are combined by the root's (member 0) finalize kernel, which reads every
 * member's accumulator over NVLink peer memory and sums the limbs as it
 * dequantizes (reduce + finalize in one pass).  The phantom is uploaded once
 * and replicated device to device (xs_ctx_copy_scene). */
typedef struct xs_group xs_group;
int xs_group_create(const int32_t* devices, int32_t n_devices, xs_group** out);
void xs_group_destroy(xs_group* grp);
int32_t xs_group_size(const xs_group* grp);
xs_context* xs_group_context(xs_group* grp, int32_t member); /* owned by the group */
const char* xs_group_last_error(const xs_group* grp);
int xs_group_set_option(xs_group* grp, const char* key, int64_t value);
int xs_group_upload_phantom(xs_group* grp, const xs_phantom* ph);
int xs_group_upload_response(xs_group* grp, const xs_response* resp);
/* REF simulate_scatter_stats, photon batches over the members. */
int xs_group_simulate_scatter_stats(xs_group* grp, const xs_geometry* g, int32_t angle_idx,
                                    const xs_spectrum* spec, const xs_sim_config* cfg,
                                    xs_scatter_result* out);
/* REF run_scan, angle ranges over the members (outputs as xs_run_scan). */
int xs_group_run_scan(xs_group* grp, const xs_geometry* g, const xs_spectrum* spec, const xs_sim_config* cfg,
                      const int32_t* angle_subset, int32_t n_subset, int32_t what, double* primary_out,
                      double* scatter_out, double* seconds_per_angle);
/* REF run_iterative_correction (as xs_run_iterative_correction on member 0)
 * with the loop's scatter and primary scans sharded by angle over the group:
 * each iteration's segmented phantom is replicated to the members device to
 * device, and their images return into member 0's stacks over NVLink. */
int xs_group_run_iterative_correction(xs_group* grp, const double* raw_intensity, const double* flatfield,
                                      const xs_geometry* g, const xs_spectrum* spec,
                                      const xs_correction_config* cfg, int32_t n_materials,
                                      const xs_material* materials, float* corrected_volume,
                                      double* corrected_stack, xs_iteration_report* reports,
                                      int32_t device_ptrs);

/* ------------------------------------------------------ files and inputs
 * The reference's file formats and text inputs (
 * csrc/files.cpp).  Same byte layouts, accepted inputs and error messages. */

/* XPRJ1 projection stack (REF detector_image.cpp:33-87): "XPRJ1", u32 nu, nv,
 * n_angles, then n_angles images of nu*nv f32.  load: images has
 * n_angles*nu*nv doubles (REF load_stack widens the f32 values);
 * save: REF save_stack narrows to f32. */
int xs_stack_file_info(const char* path, int32_t* nu, int32_t* nv, int32_t* n_angles);
int xs_stack_file_load(const char* path, double* images);
int xs_stack_file_save(const char* path, int32_t nu, int32_t nv, int32_t n_angles, const double* images);

/* XVOX1 voxel phantom (REF phantom.cpp:74-161): "XVOX1", u32 dims[3], f64
 * voxel_size[3], f64 origin[3], u32 n_materials, u8 ids, f32 densities.
 * info: REF load_phantom_header.  read: REF load_phantom's file part;
 * n_materials_given = the caller's material list length with vacuum (REF
 * fails when the header declares more); the handle owns the voxel arrays
 * its view points to (materials NULL: the caller attaches its list), and
 * xs_validate_phantom completes REF load_phantom. */
typedef struct xs_phantom_file xs_phantom_file;
int xs_phantom_file_info(const char* path, int32_t dims[3], double voxel_size[3], double origin[3],
                         uint32_t* n_materials);
int xs_phantom_file_read(const char* path, uint32_t n_materials_given, xs_phantom_file** out);
const xs_phantom* xs_phantom_file_get(const xs_phantom_file* f);
void xs_phantom_file_free(xs_phantom_file* f);
int xs_phantom_file_save(const char* path, const xs_phantom* ph);
/* REF validate_phantom (phantom.cpp:33-56) on the host (REF load_phantom runs
 * it after reading; xs_upload_phantom runs the same checks on the device). */
int xs_validate_phantom(const xs_phantom* ph);

/* XVOL1 volume (REF volume.cpp:22-62): "XVOL1", u32 dims[3], f64
 * voxel_size[3], f32 values, x fastest. */
int xs_volume_file_info(const char* path, int32_t dims[3], double voxel_size[3]);
int xs_volume_file_load(const char* path, float* values);
int xs_volume_file_save(const char* path, const int32_t dims[3], const double voxel_size[3], const float* values);

/* Material table file (REF load_material, material.cpp:129-213, with
 * validate_material :57-97); the handle owns the tables its view points to. */
typedef struct xs_material_file xs_material_file;
int xs_material_file_load(const char* path, xs_material_file** out);
const xs_material* xs_material_file_get(const xs_material_file* f);
void xs_material_file_free(xs_material_file* f);

/* Spectrum CSV (keV, weight; REF load_spectrum, spectrum.cpp:32-60). */
typedef struct xs_spectrum_file xs_spectrum_file;
int xs_spectrum_file_load(const char* path, xs_spectrum_file** out);
const xs_spectrum* xs_spectrum_file_get(const xs_spectrum_file* f);
void xs_spectrum_file_free(xs_spectrum_file* f);

/* Detector response CSV (keV, dqe, deposit_keV; REF load_detector_response,
 * detector_response.cpp:50-79). */
typedef struct xs_response_file xs_response_file;
int xs_response_file_load(const char* path, xs_response_file** out);
const xs_response* xs_response_file_get(const xs_response_file* f);
void xs_response_file_free(xs_response_file* f);

#ifdef __cplusplus
}
#endif

#endif /* XSCAT_GPU_H */
