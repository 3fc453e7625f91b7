/*
 * xscat_oracle.h — CPU oracle for the B200 projector.  TEST INFRASTRUCTURE
 * ONLY: a plain-C restatement of the reference's projector path
 * (/root/reference/proj/src/{transport,trace,cross_sections,samplers,
 * material,postprocess}.cpp).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker.  The product (libxscatgpu.so) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * reference library is compiled from /root/reference by oracle/Makefile into
 * oracle/_ref/libxscat_ref.so (same xs_* structs, see ref_capi.cpp), and the
 * tests compare both bit-for-bit plus against REF's recorded known answers
 * (tests/golden/).
 *
 * All types are the C-ABI structs of include/xscat_gpu.h.
 */
#ifndef XSCAT_ORACLE_H
#define XSCAT_ORACLE_H

#include "../include/xscat_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* xo_last_error(void);

/* Philox4x32-10 stream (REF rng.hpp:11-67): n doubles from uniform() or
 * n raw u32 from next_u32(). */
void xo_rng_uniform(uint64_t seed, uint32_t angle, uint32_t bin, uint32_t photon, int64_t n,
                    double* out);
void xo_rng_u32(uint64_t seed, uint32_t angle, uint32_t bin, uint32_t photon, int64_t n,
                uint32_t* out);

/* Table1D::loglog / linear / linear_clamped (REF table.hpp:38-69). */
int xo_table_eval(const xs_table* t, int32_t mode /*0 linear,1 clamped,2 loglog*/, double x,
                  double* y);

/* F^2 dq^2 CDF (REF material.cpp:107-125); out has f_factor.n entries. */
int xo_f2_q2_cdf(const xs_material* m, double* out);

/* Cross sections (REF cross_sections.cpp:19-96). */
int xo_p_lambda(const xs_material* m, int32_t compton, double energy_kev, double theta,
                double* p);
int xo_d_sigma(const xs_material* m, int32_t compton, double energy_kev, double theta,
               double* d);

/* Samplers (REF samplers.cpp): n draws of theta (and phi, alpha') from one
 * CounterRng(seed) stream, exactly like acceptance criterion 1. */
int xo_sample_compton(const xs_material* m, double energy_kev, uint64_t seed, int64_t n,
                      double* theta, double* phi, double* alpha_prime);
int xo_sample_rayleigh(const xs_material* m, double energy_kev, uint64_t seed, int64_t n,
                       double* theta, double* phi);
int xo_kahn_cos_theta(double alpha, uint64_t seed, int64_t n, double* cos_theta);
int xo_select_interaction(const xs_material* m, double energy_kev, uint64_t seed, int64_t n,
                          int32_t* kinds /*0 pe, 1 compton, 2 rayleigh*/);
void xo_rotate_direction(const double dir[3], double theta, double phi, double out[3]);

/* Tracing (REF trace.cpp). */
int xo_trace_attenuation(const xs_phantom* ph, const double origin[3], const double dir[3],
                         double energy_kev, int32_t step_voxels, double* tau);
int xo_trace_rho_lengths(const xs_phantom* ph, const double origin[3], const double dir[3],
                         double* rho_len /* n_materials */);
int xo_sample_free_path(const xs_phantom* ph, const double origin[3], const double dir[3],
                        double energy_kev, double u, int32_t* escaped, double point[3],
                        int32_t voxel[3]);

/* Transport (REF transport.cpp). */
int xo_apportion_photons(const xs_spectrum* spec, uint64_t photons_total, uint64_t* counts);
int xo_simulate_scatter_stats(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                              const xs_spectrum* spec, const xs_response* resp,
                              const xs_sim_config* cfg, int32_t workers, xs_scatter_result* out);
int xo_simulate_primary(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                        const xs_spectrum* spec, const xs_response* resp,
                        const xs_sim_config* cfg, int32_t workers, double* image);

/* Same histories as xo_simulate_scatter_stats, tallied into the
 * deterministic fixed-point accumulator of include/xscat_gpu.h for the
 * global history range [hist_begin, hist_end); accum is added into. */
int xo_scatter_accumulate_range(const xs_phantom* ph, const xs_geometry* g, int32_t angle_idx,
                                const xs_spectrum* spec, const xs_response* resp,
                                const xs_sim_config* cfg, uint64_t hist_begin,
                                uint64_t hist_end, uint64_t* accum);

/* Post-processing (REF postprocess.cpp), one image per call. */
int xo_sg_kernel(int32_t left, int32_t right, int32_t polyorder, double* out);
int xo_default_sg_spec(int32_t nu, int32_t nv, int32_t* window, int32_t* polyorder);
int xo_sg_smooth(const double* in, double* out, int32_t nu, int32_t nv, int32_t window,
                 int32_t polyorder);
int xo_interpolate_angles(const double* in, const double* src_angles, int32_t n_src,
                          double* out, const double* tgt_angles, int32_t n_tgt, int32_t nu,
                          int32_t nv);
int xo_upsample_image(const double* in, int32_t nu, int32_t nv, double* out, int32_t nu_out,
                      int32_t nv_out);
int xo_downsample_average(const double* in, int32_t nu, int32_t nv, double* out,
                          int32_t nu_out, int32_t nv_out);

/* Correction-loop stages (REF recon.cpp:324-348, correction.cpp:58-86, :199-246). */
int xo_intensity_to_attenuation(const double* intensity, const double* flat, int32_t nu, int32_t nv,
                                int32_t n, double* out);
int xo_correct_projections(const double* a, const double* primary, const double* scatter, int32_t nu,
                           int32_t nv, int32_t n, double* out, uint64_t* clamped);
int xo_correction_tail(const double* scatter_sub, const double* sub_angles, int32_t n_sub,
                       const double* primary_mc, const double* full_angles, int32_t n_full, int32_t nu,
                       int32_t nv, int32_t sg_window, int32_t sg_order, const double* a, int32_t nu_out,
                       int32_t nv_out, double* corrected, double* mean_fraction, uint64_t* clamped);

/* FDK (REF recon.cpp:58-157). */
int xo_fbp_reconstruct(const double* stack, const double* angles, int32_t n_views, int32_t nu, int32_t nv,
                       const xs_geometry* g, const int32_t dims[3], const double voxel[3], int32_t hann,
                       float* volume);

/* Segmentation (REF recon.cpp:159-322). */
int xo_otsu_thresholds(const float* vol, const int32_t dims[3], int32_t n_classes, int32_t bins,
                       double* thresholds);
int xo_segment_volume(const float* vol, uint64_t n, const double* thr, int32_t n_thr, int32_t n_class_map,
                      uint8_t* labels);
int xo_to_density_phantom(const uint8_t* labels, const int32_t src[3], const xs_class_spec* cls,
                          int32_t n_classes, const int32_t tgt[3], int32_t n_materials,
                          const xs_material* materials, uint8_t* ids, float* dens);

#ifdef __cplusplus
}
#endif

#endif
