// levels.cu — uniform-block levels of the device voxel grid (see
// Grid::lvl_log2 in xs_types.h), computed on the device right after the
// encoded grid is uploaded.
//
// A voxel carries the level of the largest aligned block (edges `edges[l]`,
// powers of two) that lies wholly inside the grid and holds a single palette
// code.  Passes over bricks or blocks, not voxels: brick codes, block codes
// per level (bottom-up), then every brick of a uniform block is rewritten
// with code | level << lvl_shift; an edge-2 level, if requested, marks the
// uniform 2x2x2 sub-blocks of the remaining (mixed) bricks.
#include <cstdint>

#include "xs_types.h"

namespace xsd {

namespace {

// uniform code of a brick wholly inside the grid, else -1
__global__ void brick_codes(const uint8_t* __restrict__ vox, Grid G, int bb, int16_t* __restrict__ out)
{
    const uint64_t n = (uint64_t)G.nbx * G.nby * G.nbz;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
        const int bx = (int)(b % G.nbx), by = (int)((b / G.nbx) % G.nby), bz = (int)(b / ((uint64_t)G.nbx * G.nby));
        int code = -1;
        if (4 * bx + 4 <= G.nx && 4 * by + 4 <= G.ny && 4 * bz + 4 <= G.nz) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(vox + b * bb);
            const uint32_t w0 = w[0];
            bool same = true;
            for (int i = 1; i < bb / 4; ++i)
                same &= w[i] == w0;
            same &= (w0 & 0xFFu) == ((w0 >> 8) & 0xFFu) && (w0 & 0xFFu) == ((w0 >> 16) & 0xFFu) &&
                    (w0 & 0xFFu) == (w0 >> 24);
            const int b0 = (int)(w0 & 0xFFu);
            if (same)
                code = bb == 32 ? ((b0 & 0xF) == (b0 >> 4) ? (b0 & 0xF) : -1) : b0;
        }
        out[b] = (int16_t)code;
    }
}

// uniform code of each block of f^3 children (or -1)
__global__ void block_codes(const int16_t* __restrict__ child, int cnx, int cny, int cnz, int f,
                            int16_t* __restrict__ out, int qx, int qy, int qz)
{
    const uint64_t n = (uint64_t)qx * qy * qz;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
        const int x = (int)(q % qx), y = (int)((q / qx) % qy), z = (int)(q / ((uint64_t)qx * qy));
        int code = -2;
        for (int k = 0; k < f * f * f && code != -1; ++k) {
            const int cx = x * f + k % f, cy = y * f + (k / f) % f, cz = z * f + k / (f * f);
            const int cc = (cx < cnx && cy < cny && cz < cnz) ? child[cx + (size_t)cnx * (cy + (size_t)cny * cz)] : -1;
            code = (cc < 0 || (code >= 0 && cc != code)) ? -1 : cc;
        }
        out[q] = (int16_t)(code < 0 ? -1 : code);
    }
}

struct LevelTabs {
    const int16_t* code[8];
    int nx[8], ny[8];
    int edge_b[8]; // block edge in bricks
    int n;
    int lvl0; // level number of edges[0] is lvl0 + 1
};

__global__ void rewrite_bricks(uint8_t* __restrict__ vox, Grid G, int bb, LevelTabs L)
{
    const uint64_t n = (uint64_t)G.nbx * G.nby * G.nbz;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
        const int bx = (int)(b % G.nbx), by = (int)((b / G.nbx) % G.nby), bz = (int)(b / ((uint64_t)G.nbx * G.nby));
        int level = 0, code = -1;
        for (int l = L.n - 1; l >= 0 && level == 0; --l) {
            const int e = L.edge_b[l];
            const int cc = L.code[l][bx / e + (size_t)L.nx[l] * (by / e + (size_t)L.ny[l] * (bz / e))];
            if (cc >= 0) {
                level = l + 1 + L.lvl0;
                code = cc;
            }
        }
        if (!level)
            continue;
        const int f = code | (level << G.lvl_shift);
        const uint32_t byte = bb == 32 ? (uint32_t)((f | (f << 4)) & 0xFF) : (uint32_t)(f & 0xFF);
        const uint32_t word = byte * 0x01010101u;
        uint32_t* w = reinterpret_cast<uint32_t*>(vox + b * bb);
        for (int i = 0; i < bb / 4; ++i)
            w[i] = word;
    }
}

// Edge-2 level inside mixed bricks: each uniform 2x2x2 sub-block of a brick
// that carries no larger level gets level `lvl` (voxel granularity; cell
// index inside a brick = x | y << 2 | z << 4).
__global__ void mark_subbricks(uint8_t* __restrict__ vox, Grid G, int bb, int lvl)
{
    const uint64_t n = (uint64_t)G.nbx * G.nby * G.nbz;
    const uint32_t lmask = (uint32_t)G.ubit;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n; b += (uint64_t)gridDim.x * blockDim.x) {
        const int bx = (int)(b % G.nbx), by = (int)((b / G.nbx) % G.nby), bz = (int)(b / ((uint64_t)G.nbx * G.nby));
        uint8_t* p = vox + b * bb;
        auto get = [&](int c) -> uint32_t {
            return bb == 32 ? (uint32_t)((p[c >> 1] >> ((c & 1) * 4)) & 0xF) : (uint32_t)p[c];
        };
        if (get(0) & lmask) // the brick is inside a larger uniform block
            continue;
        for (int sb = 0; sb < 8; ++sb) {
            const int x0 = 2 * (sb & 1), y0 = 2 * ((sb >> 1) & 1), z0 = 2 * (sb >> 2);
            if (4 * bx + x0 + 2 > G.nx || 4 * by + y0 + 2 > G.ny || 4 * bz + z0 + 2 > G.nz)
                continue; // padding voxels beyond the grid
            const int c0 = x0 | (y0 << 2) | (z0 << 4);
            const uint32_t code = get(c0);
            bool same = true;
            for (int k = 1; k < 8 && same; ++k)
                same = get(c0 + (k & 1) + ((k >> 1) & 1) * 4 + (k >> 2) * 16) == code;
            if (!same)
                continue;
            const uint32_t f = code | ((uint32_t)lvl << G.lvl_shift);
            for (int k = 0; k < 8; ++k) {
                const int c = c0 + (k & 1) + ((k >> 1) & 1) * 4 + (k >> 2) * 16;
                if (bb == 32) {
                    const int sh = (c & 1) * 4;
                    p[c >> 1] = (uint8_t)((p[c >> 1] & ~(0xF << sh)) | (f << sh));
                } else {
                    p[c] = (uint8_t)f;
                }
            }
        }
    }
}

// Runs (Grid::run_*), P8 only: every voxel gets the count of the voxels
// after it along the run axis, in the run direction, with the same palette
// index (capped).  Only the run bits are rewritten; a byte's palette bits,
// which the neighbours read, never change.
__global__ void run_field(uint8_t* __restrict__ vox, Grid G, int axis, int sign, int shift, int cap)
{
    const uint64_t n = (uint64_t)G.nx * G.ny * G.nz;
    const uint32_t pal = (1u << shift) - 1u;
    const uint32_t rbits = (uint32_t)cap << shift;
    const uint32_t sy = (uint32_t)G.nbx << 6, sz = (uint32_t)G.nbx * (uint32_t)G.nby << 6;
    auto cell = [&](int x, int y, int z) {
        return ((uint32_t)(x >> 2) << 6) + (uint32_t)(x & 3) + (uint32_t)(y >> 2) * sy + ((uint32_t)(y & 3) << 2) +
               (uint32_t)(z >> 2) * sz + ((uint32_t)(z & 3) << 4);
    };
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        // consecutive threads walk the run axis' neighbours (coalesced enough:
        // x-fastest order for both axes, the y run reads 4-voxel brick rows)
        const int x = (int)(v % G.nx), y = (int)((v / G.nx) % G.ny), z = (int)(v / ((uint64_t)G.nx * G.ny));
        const uint32_t c0 = cell(x, y, z);
        const uint32_t b = vox[c0];
        const uint32_t code = b & pal;
        int r = 0;
        int px = x, py = y;
        while (r < cap) {
            px += axis == 0 ? sign : 0;
            py += axis == 1 ? sign : 0;
            if ((uint32_t)px >= (uint32_t)G.nx || (uint32_t)py >= (uint32_t)G.ny)
                break;
            if ((vox[cell(px, py, z)] & pal) != code)
                break;
            ++r;
        }
        vox[c0] = (uint8_t)((b & ~rbits) | ((uint32_t)r << shift));
    }
}

} // namespace

cudaError_t launch_run_field(uint8_t* vox, const Grid& G, int axis, int sign, int shift, int cap, int sm_count,
                             cudaStream_t s)
{
    run_field<<<sm_count * 8, 256, 0, s>>>(vox, G, axis, sign, shift, cap);
    return cudaGetLastError();
}

// scratch: int16 per brick plus the (smaller) level tables; returns the
// bytes needed when scratch == nullptr
size_t levels_scratch_bytes(const Grid& G, const int* edges, int n_levels)
{
    if (n_levels > 0 && edges[0] == 2) {
        ++edges;
        --n_levels;
    }
    size_t total = (size_t)G.nbx * G.nby * G.nbz;
    int px = G.nbx, py = G.nby, pz = G.nbz, prev = 4;
    for (int l = 0; l < n_levels; ++l) {
        const int f = edges[l] / prev;
        px = (px + f - 1) / f;
        py = (py + f - 1) / f;
        pz = (pz + f - 1) / f;
        total += (size_t)px * py * pz;
        prev = edges[l];
    }
    return total * sizeof(int16_t) + 256;
}

cudaError_t launch_mark_levels(uint8_t* vox, const Grid& G, int fmt, const int* edges, int n_levels,
                               void* scratch, int sm_count, cudaStream_t s)
{
    if (n_levels <= 0)
        return cudaSuccess;
    const int bb = fmt == kFmtP4 ? 32 : 64;
    const int sub = edges[0] == 2 ? 1 : 0; // level 1 = 2x2x2 sub-blocks of mixed bricks
    edges += sub;
    n_levels -= sub;
    const int grid = sm_count * 8, block = 256;
    int16_t* bricks = static_cast<int16_t*>(scratch);
    brick_codes<<<grid, block, 0, s>>>(vox, G, bb, bricks);
    LevelTabs L{};
    L.n = n_levels;
    const int16_t* prev = bricks;
    int px = G.nbx, py = G.nby, pz = G.nbz, pe = 4;
    int16_t* next = bricks + (size_t)G.nbx * G.nby * G.nbz;
    for (int l = 0; l < n_levels; ++l) {
        const int f = edges[l] / pe;
        const int qx = (px + f - 1) / f, qy = (py + f - 1) / f, qz = (pz + f - 1) / f;
        block_codes<<<grid, block, 0, s>>>(prev, px, py, pz, f, next, qx, qy, qz);
        L.code[l] = next;
        L.nx[l] = qx;
        L.ny[l] = qy;
        L.edge_b[l] = edges[l] / 4;
        L.lvl0 = sub;
        prev = next;
        next += (size_t)qx * qy * qz;
        px = qx;
        py = qy;
        pz = qz;
        pe = edges[l];
    }
    if (n_levels > 0)
        rewrite_bricks<<<grid, block, 0, s>>>(vox, G, bb, L);
    if (sub)
        mark_subbricks<<<grid, block, 0, s>>>(vox, G, bb, 1);
    return cudaGetLastError();
}

} // namespace xsd
