// xs_types.h — POD types shared by the host launcher and the kernels.
#pragma once

#include <cstdint>

namespace xsd {

constexpr int kMaxMaterials = 8; // incl. vacuum; the REF bundle has 5
constexpr int kMaxPalette = 256;
constexpr int kMaxBins = 1024;

enum VoxelFormat : int32_t { kFmtP4 = 0, kFmtP8 = 1, kFmtRaw = 2 };

// Offsets into the packed fp64 table buffer: x[n] y[n] log x[n] log y[n].
struct TabDesc {
    int32_t off;
    int32_t n;
};

struct MatDesc {
    TabDesc mu, incoh, coh, pe; // energy tables (log-log)
    TabDesc s, f;               // form factors (linear)
    int32_t cdf_off;            // F^2 dq^2 cumulative mass (REF material.cpp:107-125)
    int32_t has_tables;
    double z_eff;
};

struct Grid {
    int32_t nx, ny, nz, nbx, nby, nbz;
    double ox, oy, oz;    // origin (low corner)
    double hx, hy, hz;    // voxel size
    double ihx, ihy, ihz; // 1 / voxel size (REF computes 1.0 / hs per call; same value)
    double ux, uy, uz;    // origin + extent (REF VoxelPhantom::extent)
    const uint8_t* vox;   // P4 nibbles / P8 codes / raw ids, bricked
    const float* dens;    // raw densities, bricked (raw format only)
    int32_t fmt;
    int32_t n_codes;      // palette size (P4/P8)
    // Uniform-block level in the palette codes: the bits above the palette
    // index (ubit = their mask, lvl_shift = their position; up to three)
    // give the level of the largest aligned uniform block (all voxels the
    // same code) holding the voxel; nibble l of lvl_log2 is log2 of that
    // block's edge (level 0: not uniform, edge 1).
    int32_t ubit;
    int32_t lvl_shift;
    uint32_t lvl_log2;
    // Runs (P8 block walk, spare bits between the palette index and the
    // level): the number of voxels after this one, along axis run_axis (0: x,
    // 1: y) in direction run_sign, that hold the same palette index, capped
    // at run_mask.  Set for the travel direction of the current projection
    // (levels.cu run_field); run_mask = 0: no runs.
    int32_t run_shift;
    int32_t run_mask;
    int32_t run_axis;
    int32_t run_sign;
    int32_t pad_;
};

// Device error record; code is an xs_status.
struct DevStatus {
    int32_t code;
    int32_t what;
    int32_t bin;
    int32_t pad;
    double energy;
    double value;
};

enum ErrWhat : int32_t {
    kErrNonFinite = 1,
    kErrTableRange = 2,
    kErrTallyOverflow = 3,
    kErrSigmaIncoh = 4,
    kErrSigmaCoh = 5,
    kErrSigmaAll = 6,
    kErrComptonS = 7,
    kErrRayleighF = 8,
    kErrTheta = 9,
    kErrStuck = 10,
};

struct TransportParams {
    Grid G;
    const double* tabs;
    int32_t n_mats;
    int32_t n_pal;
    MatDesc mats[kMaxMaterials];
    uint8_t pal_mat[kMaxPalette];
    float pal_dens[kMaxPalette];
    TabDesc resp_deposit;

    // projection frame (host-computed with glibc cos/sin, REF scan_geometry.cpp:44-67)
    double src[3], center[3], uaxis[3], normal[3];
    int32_t nu, nv;
    double pitch;
    double det_area; // REF ScanGeometry::detector_area()
    double n_pixels; // (double)nu * nv

    // spectrum
    int32_t n_bins;
    const double* bin_energy;
    const double* bin_weight;
    const uint64_t* bin_start; // n_bins + 1, global bin-major history offsets
    const uint64_t* bin_count; // photons per bin (REF apportion_photons)

    // config
    uint32_t k0, k1, angle;
    int32_t splitting;
    double survival, wmin_rel;
    int32_t step_voxels;
    int32_t max_inter;
    int32_t track_var;
    int32_t var_cap;
    double march_h;
    double march_ih; // 1 / march_h
    int32_t skip;           // 1: cross uniform macro cells in one step
    int32_t shared_mu_grid; // all materials' mu tables share grid_mat's energy knots
    int32_t shared_e_grid;  // ... and so do their sigma_incoh / sigma_coh / sigma_pe tables
    int32_t grid_mat;

    // tallies
    unsigned long long* accum;
    uint64_t off_image, off_var, off_bins, off_ledger, off_diag;
    int32_t log2_img, log2_w;

    // history range and pool
    uint64_t h_begin, h_end;
    unsigned long long* pool;
    int32_t grab;           // histories per warp grab
    int32_t slots_per_warp; // live histories per warp (<= 64)
    int32_t queue_len;      // scoring FIFO entries per warp (H * splitting + 1)

    // variance scratch: var_cap entries per history slot
    uint32_t* var_pix;
    double* var_val;

    DevStatus* status;
};

// Wavefront engine run summary (wavefront.cu).
struct WaveInfo {
    uint32_t waves;
    uint32_t n_slots;
    int32_t walk_blocks_per_sm;
    uint32_t launches;
    float walk_ms; // summed device time of the walk kernels
    float setup_ms, score_ms, event_ms, admit_ms; // XSCAT_KTIME: the other kernels (plan + admit)
};

// Angular interpolation plan entry (REF postprocess.cpp:160-192).
struct InterpEntry {
    int32_t lo, hi, exact;
    double w;
};

struct PrimaryParams {
    Grid G;
    int32_t n_mats;
    int32_t n_pal;
    uint8_t pal_mat[kMaxPalette];
    float pal_dens[kMaxPalette];
    double src[3], center[3], uaxis[3];
    int32_t nu, nv;
    double pitch;
    int32_t n_bins;
    const double* atten;    // [n_bins][n_mats] mass attenuation (host glibc loglog)
    const double* wresp;    // [n_bins] spectrum weight
    const double* response; // [n_bins] response factor
    double* image;
    DevStatus* status;
};

} // namespace xsd
