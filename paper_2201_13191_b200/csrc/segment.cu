// segment.cu — the segmentation stage of the correction loop on the device
// (SURVEY.md §8(f) rank 3): REF otsu_thresholds, segment_volume and
// to_density_phantom (recon.cpp:159-322), plus the device side of a phantom
// upload whose arrays are already in device memory (validation, palette
// discovery and brick encoding; REF validate_phantom, phantom.cpp:33-56).
//
// Together they build the next iteration's scatter phantom from the FDK
// volume without leaving HBM (REF correction.cpp:167-172).  Everything is
// exact: min / max and integer histogram counts do not depend on the order
// of the reduction, the dynamic programme and the block means run in REF's
// order inside one thread, so thresholds, labels and phantoms are
// bit-identical to REF.
#include <cstddef>
#include <cstdint>

#include "xs_types.h"

namespace xsd {

// Device record shared by the segmentation kernels (one per context).
struct SegCtl {
    uint32_t lo_key, hi_key;         // ordered-float keys of the interior min / max
    unsigned long long first_bad;    // smallest offending voxel index (validation / labels)
    uint32_t n_pairs, overflow;      // distinct (id, density) pairs seen
    int32_t status;                  // 0 ok, 1 degenerate histogram
    int32_t pad;
    double lo, hi, scale;
    unsigned long long hash[1024];   // (id << 32 | density bits), ~0 = empty
};
// capi.cu reads the record through these offsets (SegCtlView)
static_assert(offsetof(SegCtl, first_bad) == 8 && offsetof(SegCtl, n_pairs) == 16 &&
                  offsetof(SegCtl, overflow) == 20 && offsetof(SegCtl, status) == 24 &&
                  offsetof(SegCtl, lo) == 32 && offsetof(SegCtl, hash) == 56,
              "SegCtl layout");

namespace {

constexpr int kThr = 256;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr unsigned long long kEmpty = ~0ull;

// Float -> unsigned key with the same order (NaN excluded by the caller).
__device__ __forceinline__ uint32_t fkey(float v)
{
    const uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float kfloat(uint32_t k)
{
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

struct Interior {
    int x0, y0, z0, nx, ny, nz; // box [x0, x0 + nx) ...
    int dx, dy;                 // volume row / plane strides
};

__device__ __forceinline__ uint64_t interior_index(const Interior& I, uint64_t i)
{
    const uint64_t x = i % (uint64_t)I.nx, r = i / (uint64_t)I.nx;
    const uint64_t y = r % (uint64_t)I.ny, z = r / (uint64_t)I.ny;
    return (uint64_t)(I.x0 + x) + (uint64_t)I.dx * ((uint64_t)(I.y0 + y) + (uint64_t)I.dy * (uint64_t)(I.z0 + z));
}

// REF recon.cpp:167-178: interior min / max (NaN never replaces lo / hi there).
__global__ void __launch_bounds__(kThr) otsu_minmax(const float* __restrict__ vol, Interior I, SegCtl* ctl)
{
    const uint64_t n = (uint64_t)I.nx * I.ny * I.nz;
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = vol[interior_index(I, i)];
        if (v == v) {
            const uint32_t k = fkey(v);
            lo = min(lo, k);
            hi = max(hi, k);
        }
    }
    lo = __reduce_min_sync(kFull, lo);
    hi = __reduce_max_sync(kFull, hi);
    if ((threadIdx.x & 31) == 0) {
        if (lo != 0xFFFFFFFFu)
            atomicMin(&ctl->lo_key, lo);
        if (hi != 0u)
            atomicMax(&ctl->hi_key, hi);
    }
}

__device__ __forceinline__ bool otsu_range(SegCtl* ctl, int bins, double& lo, double& scale)
{
    if (ctl->lo_key == 0xFFFFFFFFu)
        return false; // all NaN: lo = +inf, hi = -inf in REF
    lo = (double)kfloat(ctl->lo_key);
    const double hi = (double)kfloat(ctl->hi_key);
    if (!(hi > lo))
        return false;
    scale = bins / (hi - lo);
    return true;
}

// REF recon.cpp:180-190: b = clamp(int((v - lo) * scale), 0, bins - 1).
// (int) of NaN is bin 0 here and, through clamp(INT_MIN), in REF.
__global__ void __launch_bounds__(kThr) otsu_hist(const float* __restrict__ vol, Interior I, int bins, SegCtl* ctl,
                                                  unsigned* __restrict__ count, int use_smem)
{
    extern __shared__ unsigned sh[];
    double lo, scale;
    if (!otsu_range(ctl, bins, lo, scale))
        return;
    unsigned* h = use_smem ? sh : count;
    if (use_smem) {
        for (int b = threadIdx.x; b < bins; b += blockDim.x)
            sh[b] = 0u;
        __syncthreads();
    }
    const uint64_t n = (uint64_t)I.nx * I.ny * I.nz;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double v = (double)vol[interior_index(I, i)];
        int b = __double2int_rz(__dmul_rn(__dsub_rn(v, lo), scale));
        b = b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
        atomicAdd(h + b, 1u);
    }
    if (use_smem) {
        __syncthreads();
        for (int b = threadIdx.x; b < bins; b += blockDim.x)
            if (sh[b])
                atomicAdd(count + b, sh[b]);
    }
}

// REF recon.cpp:192-239: prefix sums, the exact dynamic programme over
// (class, last bin), backtracking, thresholds lo + cut / scale.  One block;
// thread b owns best[k][b] and scans m in REF's order with REF's strict '>'.
__global__ void __launch_bounds__(1024) otsu_dp(const unsigned* __restrict__ count, int bins, int n_classes,
                                                double* __restrict__ pc, double* __restrict__ ps,
                                                double* __restrict__ best, int* __restrict__ arg, SegCtl* ctl,
                                                double* __restrict__ thresholds)
{
    double lo, scale;
    const bool ok = otsu_range(ctl, bins, lo, scale);
    if (!ok) {
        if (threadIdx.x == 0)
            ctl->status = 1;
        return;
    }
    const double neg_inf = __longlong_as_double((long long)0xFFF0000000000000ull);
    const int W = bins + 1;
    if (threadIdx.x == 0) {
        pc[0] = 0.0;
        ps[0] = 0.0;
        for (int b = 0; b < bins; ++b) {
            const double c = (double)count[b];
            pc[b + 1] = __dadd_rn(pc[b], c);
            ps[b + 1] = __dadd_rn(ps[b], __dmul_rn(c, (double)b + 0.5));
        }
    }
    for (int i = threadIdx.x; i < (n_classes + 1) * W; i += blockDim.x) {
        best[i] = neg_inf;
        arg[i] = -1;
    }
    __syncthreads();
    if (threadIdx.x == 0)
        best[0] = 0.0;
    __syncthreads();
    for (int k = 1; k <= n_classes; ++k) {
        for (int b = k + threadIdx.x; b <= bins; b += blockDim.x) {
            double bb = neg_inf;
            int am = -1;
            const double pcb = pc[b], psb = ps[b];
            for (int m = k - 1; m < b; ++m) {
                const double prev = best[(k - 1) * W + m];
                if (prev == neg_inf)
                    continue;
                const double n = __dsub_rn(pcb, pc[m]);
                double sc;
                if (n <= 0.0) {
                    sc = neg_inf;
                } else {
                    const double s = __dsub_rn(psb, ps[m]);
                    sc = __ddiv_rn(__dmul_rn(s, s), n);
                }
                const double cand = __dadd_rn(prev, sc);
                if (cand > bb) {
                    bb = cand;
                    am = m;
                }
            }
            best[k * W + b] = bb;
            arg[k * W + b] = am;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (best[n_classes * W + bins] == neg_inf) {
            ctl->status = 1;
            return;
        }
        int cuts[4];
        int b = bins;
        for (int k = n_classes; k >= 1; --k) {
            cuts[k - 1] = arg[k * W + b]; // ascending after the leading 0 is dropped
            b = arg[k * W + b];
        }
        for (int k = 1; k < n_classes; ++k)
            thresholds[k - 1] = __dadd_rn(lo, __ddiv_rn((double)cuts[k], scale));
        ctl->lo = lo;
        ctl->scale = scale;
        ctl->status = 0;
    }
}

// REF recon.cpp:255-260.
__device__ __forceinline__ int label_of(double v, const double* thr, int n_thr)
{
    int label = 0;
    while (label < n_thr && v >= thr[label])
        ++label;
    return label;
}

__global__ void __launch_bounds__(kThr) segment_labels(const float* __restrict__ vol, uint64_t n,
                                                       const double* __restrict__ thr_g, int n_thr,
                                                       uint8_t* __restrict__ labels)
{
    __shared__ double thr[256];
    for (int i = threadIdx.x; i < n_thr; i += blockDim.x)
        thr[i] = thr_g[i];
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        labels[i] = (uint8_t)label_of((double)vol[i], thr, n_thr);
}

struct DensArgs {
    int sx, sy, sz; // source (volume) dims
    int tx, ty, tz; // target dims
    int n_labels;
    int n_thr;
    int cls_mat[16];
    double cls_dens[16];
    double thr[15];
};

// REF recon.cpp:264-322 (after its label check): per output voxel the modal
// label of its block (ties to the higher label) and the block mean of the
// class densities, summed in REF's (z, y, x) order.  FROM_VOLUME: labels
// computed inline from the volume and the thresholds (segment_volume fused).
template <bool FROM_VOLUME>
__global__ void __launch_bounds__(kThr) density_phantom(const uint8_t* __restrict__ labels,
                                                        const float* __restrict__ vol, const DensArgs A,
                                                        uint8_t* __restrict__ id_out, float* __restrict__ dens_out,
                                                        SegCtl* ctl)
{
    const uint64_t n = (uint64_t)A.tx * A.ty * A.tz;
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < n; o += (uint64_t)gridDim.x * blockDim.x) {
        const int ox = (int)(o % A.tx), oy = (int)((o / A.tx) % A.ty), oz = (int)(o / ((uint64_t)A.tx * A.ty));
        const int z0 = (int)((int64_t)oz * A.sz / A.tz), z1 = (int)((int64_t)(oz + 1) * A.sz / A.tz);
        const int y0 = (int)((int64_t)oy * A.sy / A.ty), y1 = (int)((int64_t)(oy + 1) * A.sy / A.ty);
        const int x0 = (int)((int64_t)ox * A.sx / A.tx), x1 = (int)((int64_t)(ox + 1) * A.sx / A.tx);
        uint32_t votes[16];
#pragma unroll
        for (int l = 0; l < 16; ++l)
            votes[l] = 0u;
        double rho_sum = 0.0;
        uint64_t cnt = 0;
        bool bad = false;
        for (int iz = z0; iz < z1; ++iz)
            for (int iy = y0; iy < y1; ++iy)
                for (int ix = x0; ix < x1; ++ix) {
                    const uint64_t src = (uint64_t)ix + (uint64_t)A.sx * ((uint64_t)iy + (uint64_t)A.sy * iz);
                    int label;
                    if (FROM_VOLUME)
                        label = label_of((double)vol[src], A.thr, A.n_thr);
                    else
                        label = labels[src];
                    if (label >= A.n_labels) {
                        atomicMin(&ctl->first_bad, (unsigned long long)src);
                        bad = true;
                        continue;
                    }
#pragma unroll
                    for (int l = 0; l < 16; ++l)
                        votes[l] += (l == label) ? 1u : 0u;
                    rho_sum = __dadd_rn(rho_sum, A.cls_dens[label]);
                    ++cnt;
                }
        if (bad)
            continue;
        int mode = 0;
#pragma unroll
        for (int l = 1; l < 16; ++l)
            if (l < A.n_labels && votes[l] >= votes[mode])
                mode = l;
        if (A.cls_mat[mode] == 0) {
            id_out[o] = 0;
            dens_out[o] = 0.0f;
        } else {
            id_out[o] = (uint8_t)A.cls_mat[mode];
            dens_out[o] = __double2float_rn(__ddiv_rn(rho_sum, (double)cnt));
        }
    }
}

// ------------------------------------------------ device phantom upload
// REF validate_phantom (phantom.cpp:42-54) per voxel, and the distinct
// (material, density) pairs in a small open-addressing set.
struct ScanArgs {
    uint64_t n;
    int n_materials;
    uint32_t has_tables; // bit m: material m has tables
};

__device__ __forceinline__ bool voxel_ok(uint8_t id, float d, const ScanArgs& S)
{
    if (id >= S.n_materials)
        return false;
    if (id != 0 && !((S.has_tables >> id) & 1u))
        return false;
    if (!(d >= 0.0f))
        return false;
    if (id == 0 && d != 0.0f)
        return false;
    return true;
}

__device__ __forceinline__ void pair_insert(SegCtl* ctl, unsigned long long key)
{
    if (ctl->overflow)
        return;
    uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 54); // 10 bits
    for (int probe = 0; probe < 1024; ++probe) {
        const unsigned long long cur = ((volatile unsigned long long*)ctl->hash)[h];
        if (cur == key)
            return;
        if (cur == kEmpty) {
            const unsigned long long prev = atomicCAS(&ctl->hash[h], kEmpty, key);
            if (prev == kEmpty) {
                if (atomicAdd(&ctl->n_pairs, 1u) >= (uint32_t)kMaxPalette)
                    ctl->overflow = 1;
                return;
            }
            if (prev == key)
                return;
        }
        h = (h + 1) & 1023u;
    }
    ctl->overflow = 1;
}

__global__ void __launch_bounds__(kThr) phantom_scan(const uint8_t* __restrict__ ids, const float* __restrict__ dens,
                                                     ScanArgs S, SegCtl* ctl)
{
    unsigned long long last = kEmpty;
    // warp-uniform trip count: the key matching below runs with every lane of
    // the warp at the same loop iteration (full mask, no __activemask())
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); i0 < S.n; i0 += stride) {
        const uint64_t i = i0 + (threadIdx.x & 31u);
        unsigned long long key = kEmpty; // (never a real key: ids are < 2^8)
        if (i < S.n) {
            const uint8_t id = ids[i];
            const float d = dens[i];
            if (!voxel_ok(id, d, S))
                atomicMin(&ctl->first_bad, (unsigned long long)i);
            else
                key = ((unsigned long long)id << 32) | __float_as_uint(d);
        }
        const bool fresh = key != kEmpty && key != last;
        if (key != kEmpty)
            last = key;
        // one insert per distinct key of the warp
        const unsigned m = __match_any_sync(0xffffffffu, fresh ? key : kEmpty);
        if (fresh && (threadIdx.x & 31) == __ffs(m) - 1)
            pair_insert(ctl, key);
    }
}

// Brick encoding (the device twin of capi.cu encode_phantom): one thread per
// 4-voxel row of a brick; codes = index of the voxel's pair in the sorted
// palette; padding voxels get code 0 (raw: id 0, density 0).
struct EncArgs {
    int nx, ny, nz, nbx, nby, nbz;
    int fmt;
    int n_pal;
};

__global__ void __launch_bounds__(kThr) phantom_encode(const uint8_t* __restrict__ ids, const float* __restrict__ dens,
                                                       const unsigned long long* __restrict__ pal_g, EncArgs E,
                                                       uint8_t* __restrict__ vox, float* __restrict__ vdens)
{
    __shared__ unsigned long long pal[kMaxPalette];
    for (int i = threadIdx.x; i < E.n_pal; i += blockDim.x)
        pal[i] = pal_g[i];
    __syncthreads();
    const uint64_t n_rows = (uint64_t)E.nbx * (4ull * E.nby) * (4ull * E.nbz);
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_rows; r += (uint64_t)gridDim.x * blockDim.x) {
        const int bx = (int)(r % E.nbx);
        const uint64_t yz = r / E.nbx;
        const int y = (int)(yz % (4ull * E.nby)), z = (int)(yz / (4ull * E.nby));
        const uint64_t brick = (uint64_t)bx + (uint64_t)E.nbx * ((uint64_t)(y >> 2) + (uint64_t)E.nby * (z >> 2));
        const uint32_t row = (uint32_t)(((y & 3) << 2) | ((z & 3) << 4)); // cell of x & 3 == 0
        uint32_t codes = 0u;
        float dv[4] = {0.f, 0.f, 0.f, 0.f};
        uint8_t iv[4] = {0, 0, 0, 0};
        if (y < E.ny && z < E.nz) {
            for (int j = 0; j < 4; ++j) {
                const int x = 4 * bx + j;
                if (x >= E.nx)
                    break;
                const uint64_t src = (uint64_t)x + (uint64_t)E.nx * ((uint64_t)y + (uint64_t)E.ny * z);
                const uint8_t id = ids[src];
                const float d = dens[src];
                if (E.fmt == kFmtRaw) {
                    iv[j] = id;
                    dv[j] = d;
                    continue;
                }
                const unsigned long long key = ((unsigned long long)id << 32) | __float_as_uint(d);
                int lo = 0, hi = E.n_pal; // lower_bound
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (pal[mid] < key)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                codes |= (uint32_t)lo << (8 * j);
            }
        }
        const uint64_t cell = (brick << 6) | row;
        if (E.fmt == kFmtP8) {
            *reinterpret_cast<uint32_t*>(vox + cell) = codes;
        } else if (E.fmt == kFmtP4) {
            const uint16_t packed = (uint16_t)((codes & 0xFu) | (((codes >> 8) & 0xFu) << 4) |
                                               (((codes >> 16) & 0xFu) << 8) | (((codes >> 24) & 0xFu) << 12));
            *reinterpret_cast<uint16_t*>(vox + (cell >> 1)) = packed;
        } else {
            *reinterpret_cast<uint32_t*>(vox + cell) =
                (uint32_t)iv[0] | ((uint32_t)iv[1] << 8) | ((uint32_t)iv[2] << 16) | ((uint32_t)iv[3] << 24);
            *reinterpret_cast<float4*>(vdens + cell) = make_float4(dv[0], dv[1], dv[2], dv[3]);
        }
    }
}

__global__ void seg_reset(SegCtl* ctl)
{
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
        ctl->hash[i] = kEmpty;
    if (threadIdx.x == 0) {
        ctl->lo_key = 0xFFFFFFFFu;
        ctl->hi_key = 0u;
        ctl->first_bad = kEmpty;
        ctl->n_pairs = 0;
        ctl->overflow = 0;
        ctl->status = 0;
    }
}

int grid_for(uint64_t n, int sm_count)
{
    const uint64_t want = (n + kThr - 1) / kThr;
    const uint64_t cap = (uint64_t)sm_count * 8;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

// Normalised cross-correlation of two float volumes (REF metrics.cpp:19-35,
// the loop's ncc_to_previous report): two passes (means, then centred
// moments) with per-block fp64 partials over a fixed grid, combined in block
// order by one thread, so the value does not depend on the schedule.
constexpr int kNccBlocks = 592;

__device__ __forceinline__ void block_sum3(double& a, double& b, double& c)
{
    __shared__ double sh[3][kThr];
    sh[0][threadIdx.x] = a;
    sh[1][threadIdx.x] = b;
    sh[2][threadIdx.x] = c;
    __syncthreads();
    for (int s = kThr / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
            sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
            sh[2][threadIdx.x] += sh[2][threadIdx.x + s];
        }
        __syncthreads();
    }
    a = sh[0][0];
    b = sh[1][0];
    c = sh[2][0];
}

__global__ void __launch_bounds__(kThr) ncc_pass(const float* __restrict__ x1, const float* __restrict__ x2, uint64_t n,
                                                 const double* __restrict__ means, double* __restrict__ partial)
{
    double a = 0.0, b = 0.0, c = 0.0;
    const bool centred = means != nullptr;
    const double m1 = centred ? means[0] : 0.0, m2 = centred ? means[1] : 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double u = (double)x1[i] - m1, v = (double)x2[i] - m2;
        if (centred) {
            a += u * v;
            b += u * u;
            c += v * v;
        } else {
            a += u;
            b += v;
        }
    }
    block_sum3(a, b, c);
    if (threadIdx.x == 0) {
        partial[3 * blockIdx.x + 0] = a;
        partial[3 * blockIdx.x + 1] = b;
        partial[3 * blockIdx.x + 2] = c;
    }
}

__global__ void ncc_combine(const double* __restrict__ partial, int n_blocks, uint64_t n, double* __restrict__ out,
                            int final_pass)
{
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = 0; i < n_blocks; ++i) {
        a += partial[3 * i + 0];
        b += partial[3 * i + 1];
        c += partial[3 * i + 2];
    }
    if (!final_pass) { // means
        out[0] = a / (double)n;
        out[1] = b / (double)n;
    } else { // cov, v1, v2
        out[2] = a;
        out[3] = b;
        out[4] = c;
    }
}

} // namespace

size_t ncc_scratch_bytes() { return (3 * (size_t)kNccBlocks + 8) * sizeof(double); }

// out[0..4] = mean1, mean2, cov, var1, var2 (device); ncc = cov / sqrt(v1 v2)
cudaError_t launch_ncc(const float* x1, const float* x2, uint64_t n, void* scratch, cudaStream_t s)
{
    double* out = static_cast<double*>(scratch);
    double* partial = out + 8;
    ncc_pass<<<kNccBlocks, kThr, 0, s>>>(x1, x2, n, nullptr, partial);
    ncc_combine<<<1, 1, 0, s>>>(partial, kNccBlocks, n, out, 0);
    ncc_pass<<<kNccBlocks, kThr, 0, s>>>(x1, x2, n, out, partial);
    ncc_combine<<<1, 1, 0, s>>>(partial, kNccBlocks, n, out, 1);
    return cudaGetLastError();
}

size_t seg_ctl_bytes() { return sizeof(SegCtl); }

size_t otsu_scratch_bytes(int bins, int n_classes)
{
    const size_t W = (size_t)bins + 1;
    return (size_t)bins * 4 + 2 * W * 8 + (size_t)(n_classes + 1) * W * (8 + 4) + 64;
}

cudaError_t launch_seg_reset(void* ctl, cudaStream_t s)
{
    seg_reset<<<1, 256, 0, s>>>(static_cast<SegCtl*>(ctl));
    return cudaGetLastError();
}

// REF recon.cpp:159-240.  Thresholds (n_classes - 1 doubles) into `thr`;
// ctl->status = 1 for REF's "degenerate histogram".
cudaError_t launch_otsu(const float* vol, const int dims[3], int n_classes, int bins, void* ctl_, void* scratch,
                        double* thr, int sm_count, cudaStream_t s)
{
    SegCtl* ctl = static_cast<SegCtl*>(ctl_);
    auto margin = [](int n) { return n / 20 > 0 ? n / 20 : 0; };
    Interior I;
    const int mx = margin(dims[0]), my = margin(dims[1]), mz = margin(dims[2]);
    I.x0 = mx;
    I.y0 = my;
    I.z0 = mz;
    I.nx = dims[0] - 2 * mx;
    I.ny = dims[1] - 2 * my;
    I.nz = dims[2] - 2 * mz;
    I.dx = dims[0];
    I.dy = dims[1];
    const uint64_t n = (uint64_t)I.nx * I.ny * I.nz;
    const size_t W = (size_t)bins + 1;
    unsigned* count = static_cast<unsigned*>(scratch);
    double* pc = reinterpret_cast<double*>(static_cast<char*>(scratch) + (((size_t)bins * 4 + 15) & ~(size_t)15));
    double* ps = pc + W;
    double* best = ps + W;
    int* arg = reinterpret_cast<int*>(best + (size_t)(n_classes + 1) * W);
    cudaError_t e = cudaMemsetAsync(count, 0, (size_t)bins * 4, s);
    if (e != cudaSuccess)
        return e;
    const int grid = grid_for(n, sm_count);
    otsu_minmax<<<grid, kThr, 0, s>>>(vol, I, ctl);
    const int use_smem = bins <= 12 * 1024 ? 1 : 0;
    otsu_hist<<<grid, kThr, use_smem ? (size_t)bins * 4 : 0, s>>>(vol, I, bins, ctl, count, use_smem);
    otsu_dp<<<1, 1024, 0, s>>>(count, bins, n_classes, pc, ps, best, arg, ctl, thr);
    return cudaGetLastError();
}

cudaError_t launch_segment_labels(const float* vol, uint64_t n, const double* thr, int n_thr, uint8_t* labels,
                                  int sm_count, cudaStream_t s)
{
    segment_labels<<<grid_for(n, sm_count), kThr, 0, s>>>(vol, n, thr, n_thr, labels);
    return cudaGetLastError();
}

// labels != nullptr: REF to_density_phantom on given labels; else labels
// computed from `vol` and the thresholds (host copies in `thr`).
cudaError_t launch_density_phantom(const uint8_t* labels, const float* vol, const int src[3], const int tgt[3],
                                   const int* cls_mat, const double* cls_dens, int n_labels, const double* thr,
                                   int n_thr, uint8_t* id_out, float* dens_out, void* ctl, int sm_count,
                                   cudaStream_t s)
{
    DensArgs A{};
    A.sx = src[0];
    A.sy = src[1];
    A.sz = src[2];
    A.tx = tgt[0];
    A.ty = tgt[1];
    A.tz = tgt[2];
    A.n_labels = n_labels;
    A.n_thr = n_thr;
    for (int l = 0; l < n_labels && l < 16; ++l) {
        A.cls_mat[l] = cls_mat[l];
        A.cls_dens[l] = cls_dens[l];
    }
    for (int t = 0; t < n_thr && t < 15; ++t)
        A.thr[t] = thr[t];
    const uint64_t n = (uint64_t)tgt[0] * tgt[1] * tgt[2];
    if (labels)
        density_phantom<false><<<grid_for(n, sm_count), kThr, 0, s>>>(labels, vol, A, id_out, dens_out,
                                                                       static_cast<SegCtl*>(ctl));
    else
        density_phantom<true><<<grid_for(n, sm_count), kThr, 0, s>>>(labels, vol, A, id_out, dens_out,
                                                                      static_cast<SegCtl*>(ctl));
    return cudaGetLastError();
}

cudaError_t launch_phantom_scan(const uint8_t* ids, const float* dens, uint64_t n, int n_materials,
                                uint32_t has_tables, void* ctl, int sm_count, cudaStream_t s)
{
    ScanArgs S{n, n_materials, has_tables};
    phantom_scan<<<grid_for(n, sm_count), kThr, 0, s>>>(ids, dens, S, static_cast<SegCtl*>(ctl));
    return cudaGetLastError();
}

cudaError_t launch_phantom_encode(const uint8_t* ids, const float* dens, const unsigned long long* pal, int n_pal,
                                  const Grid& G, int fmt, uint8_t* vox, float* vdens, int sm_count, cudaStream_t s)
{
    EncArgs E{G.nx, G.ny, G.nz, G.nbx, G.nby, G.nbz, fmt, n_pal};
    const uint64_t rows = (uint64_t)G.nbx * 4ull * G.nby * 4ull * G.nbz;
    phantom_encode<<<grid_for(rows, sm_count), kThr, 0, s>>>(ids, dens, pal, E, vox, vdens);
    return cudaGetLastError();
}

} // namespace xsd
