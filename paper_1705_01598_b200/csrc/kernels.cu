// kernels.cu -- sm_100a kernels of the permutation hot path and their launch.
//
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
//
//   copy_kernel   rank 1 after fusion (identity), 128-bit grid-stride copy.
//   tile_kernel   generic staged tile (Tiled / Packed / PackedSplit classes,
//                 P:L121-161): per-thread loop-invariant minor offsets
//                 (Eqs. 4-6, the nReg register arrays of P:L155-159),
//                 warp-parallel major-offset decode (Algorithm 1),
//                 double-buffered shared memory with the next tile's loads in
//                 flight while the current tile is written, persistent CTAs.
//
// Elements are opaque 32/64-bit words: no float types anywhere (bit-exact).
#include <cuda_runtime.h>

#include <cstdint>

#include "tt_internal.h"

namespace tt {

// ---------------------------------------------------------------------------
// copy (row a-9, identity): 16-byte vectors when both pointers allow it
// ---------------------------------------------------------------------------
template <typename W>
__global__ void __launch_bounds__(1024) copy_kernel(const W* __restrict__ in, W* __restrict__ out,
                                                    int64_t n, int vec16) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (vec16) {
        constexpr int PER = 16 / sizeof(W);
        const int64_t n16 = n / PER;
        const uint4* __restrict__ a = reinterpret_cast<const uint4*>(in);
        uint4* __restrict__ b = reinterpret_cast<uint4*>(out);
        int64_t i = tid;
        for (; i + 3 * nthr < n16; i += 4 * nthr) {
            uint4 x0 = __ldcs(a + i);
            uint4 x1 = __ldcs(a + i + nthr);
            uint4 x2 = __ldcs(a + i + 2 * nthr);
            uint4 x3 = __ldcs(a + i + 3 * nthr);
            __stcs(b + i, x0);
            __stcs(b + i + nthr, x1);
            __stcs(b + i + 2 * nthr, x2);
            __stcs(b + i + 3 * nthr, x3);
        }
        for (; i < n16; i += nthr) __stcs(b + i, __ldcs(a + i));
        done = n16 * PER;
    }
    for (int64_t i = done + tid; i < n; i += nthr) out[i] = in[i];
}

// ---------------------------------------------------------------------------
// generic staged tile
// ---------------------------------------------------------------------------
template <typename I>
struct TileBase {
    I in, out;
    uint32_t mask;   // slot-word bits that must be set for a slot to be valid
};

// Algorithm 1: lane i < h evaluates the i-th term of Eqs. (2)
// and (3) for the tile index b = t -- mod(floor(t / c_i), d_i) * stride_i --
// and an XOR butterfly sums the terms; every lane ends with both bases.  The
// same decode order serves both sums (reading R3).  A lane holding
// a split dim also reports whether this tile is that dim's ragged last chunk
// (PackedSplit edge), gathered with one ballot.
template <typename I, typename P>
__device__ __forceinline__ TileBase<I> decode_tile(const P& p, I t, int lane) {
    I vin = 0, vout = 0;
    bool ragged = false;
    if (lane < p.h) {
        const I d = (I)p.gD[lane];
        const I q = (t / (I)p.gC[lane]) % d;
        vin = q * (I)p.gSin[lane];
        vout = q * (I)p.gSout[lane];
        ragged = (q == d - 1) &&
                 ((p.nSplit > 0 && lane == p.splitLane[0] && p.splitTail[0] != p.splitChunk[0]) ||
                  (p.nSplit > 1 && lane == p.splitLane[1] && p.splitTail[1] != p.splitChunk[1]));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        vin += __shfl_xor_sync(0xffffffffu, vin, o);
        vout += __shfl_xor_sync(0xffffffffu, vout, o);
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, ragged);
    uint32_t m = 0;
    if (p.nSplit > 0) m |= ((bal >> p.splitLane[0]) & 1u) << 14;
    if (p.nSplit > 1) m |= ((bal >> p.splitLane[1]) & 1u) << 15;
    TileBase<I> b;
    b.in = vin;
    b.out = vout;
    b.mask = m;
    return b;
}

// Slot word (one register per slot): bits 0-13 staging position of the load
// element, bit 14/15 "load element lies inside the ragged last chunk of split
// dim A/B", bits 16-29 staging position of the store element, bits 30/31 the
// same flags for it.  A slot is valid in a tile iff (word & mask) == mask.
template <typename W, int NREG, typename I>
__global__ void __launch_bounds__(512, (sizeof(I) == 8 ? 1 : 2))
tile_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    W* const sm = reinterpret_cast<W*>(smem_raw);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;

    // Per-thread loop-invariant minor positions (Eqs. 4-6; the
    // register arrays of P:L155-159): slot r handles tile element k = tid + r*NT
    // in input order (load) and k' = k in output order (store).
    I gin[NREG], gout[NREG];
    uint32_t slot[NREG];
    const int nmine = (p.V > tid) ? min(NREG, (p.V - tid + NT - 1) / NT) : 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        gin[r] = 0;
        gout[r] = 0;
        slot[r] = 0;
        if (r < nmine) {
            const int k = tid + r * NT;
            // Eq. (4): pMinorIn(k), tile-input order
            int rem = k;
            I off = 0;
            uint32_t w = 0;
            for (int i = 0; i < p.a; ++i) {
                const int c = rem % p.tExt[i];
                rem /= p.tExt[i];
                off += (I)c * (I)p.tSin[i];
                if (p.nSplit > 0 && i == p.splitTile[0] && c < p.splitTail[0]) w |= 1u << 14;
                if (p.nSplit > 1 && i == p.splitTile[1] && c < p.splitTail[1]) w |= 1u << 15;
            }
            gin[r] = off;
            w |= (uint32_t)(k + (k / p.padEvery) * p.pad);
            // Eqs. (5), (6): pMinorOut(k') and pSh(k'), tile-output order
            rem = k;
            off = 0;
            int sh = 0;
            for (int jj = 0; jj < p.a; ++jj) {
                const int t = p.tOutOrder[jj];
                const int c = rem % p.tExt[t];
                rem /= p.tExt[t];
                off += (I)c * (I)p.tSout[t];
                sh += c * p.tCin[t];
                if (p.nSplit > 0 && t == p.splitTile[0] && c < p.splitTail[0]) w |= 1u << 30;
                if (p.nSplit > 1 && t == p.splitTile[1] && c < p.splitTail[1]) w |= 1u << 31;
            }
            gout[r] = off;
            w |= (uint32_t)(sh + (sh / p.padEvery) * p.pad) << 16;
            slot[r] = w;
        }
    }

    const I nTiles = (I)p.nTiles;
    I t = (I)blockIdx.x;
    if (t >= nTiles) return;
    const I stride = (I)gridDim.x;

    W v[NREG];
    TileBase<I> cur = decode_tile<I>(p, t, lane);
#pragma unroll
    for (int r = 0; r < NREG; ++r)
        if (r < nmine && (slot[r] & cur.mask) == cur.mask) v[r] = __ldg(in + (cur.in + gin[r]));

    int buf = 0;
    for (; t < nTiles; t += stride) {
        W* const sb = sm + buf * p.sbuf;
        // stage the tile in input order
#pragma unroll
        for (int r = 0; r < NREG; ++r)
            if (r < nmine) sb[slot[r] & 0x3fffu] = v[r];
        __syncthreads();
        // issue the next tile's global loads before writing this one
        const I outBase = cur.out;
        const uint32_t omask = cur.mask << 16;
        const I tn = t + stride;
        if (tn < nTiles) {
            cur = decode_tile<I>(p, tn, lane);
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (r < nmine && (slot[r] & cur.mask) == cur.mask) v[r] = __ldg(in + (cur.in + gin[r]));
        }
        // transposed read of shared memory (Eq. 6), coalesced writes (Eq. 5)
#pragma unroll
        for (int r = 0; r < NREG; ++r)
            if (r < nmine && (slot[r] & omask) == omask)
                out[outBase + gout[r]] = sb[(slot[r] >> 16) & 0x3fffu];
        buf ^= 1;
        // Two buffers: the next iteration writes the other buffer, whose
        // readers (previous tile) all passed this iteration's barrier.
    }
}

// ---------------------------------------------------------------------------
// vectorised 2-D tiled transpose (Tiled class)
// ---------------------------------------------------------------------------
template <typename W, int VW> struct VecOf;
template <> struct VecOf<uint32_t, 4> { typedef uint4 T; };
template <> struct VecOf<uint32_t, 2> { typedef uint2 T; };
template <> struct VecOf<uint32_t, 1> { typedef uint32_t T; };
template <> struct VecOf<uint64_t, 2> { typedef ulonglong2 T; };
template <> struct VecOf<uint64_t, 1> { typedef unsigned long long T; };

// A 256-thread CTA is a 16 x 16 grid of threads; each thread owns MA x MB
// micro-tiles of VW x VW elements (MA along A, MB along B), so a tile is
// TA = 16*VW*MA (along A, the input's contiguous dim) by TB = 16*VW*MB (along
// B, the output's contiguous dim).
//   load : VW vector loads per micro-tile, lanes adjacent along A (coalesced,
//          16 lanes x VW*E bytes contiguous per row and per ma);
//   regs : VW x VW transpose in registers;
//   smem : output-major rows of TB elements in VW-element chunks, chunk index
//          XOR-swizzled by the row's micro-tile index (the bank-conflict fix of
//          P:L123's L x (L+1) padding, without the padding);
//   store: whole chunks, lanes adjacent along B (coalesced).
// Double-buffered: the next tile's loads are in flight during the stores.
template <typename W, int VW, int MA, int MB, typename I>
__global__ void __launch_bounds__(256)
tiled2d_kernel(const __grid_constant__ Tiled2DParams p, const W* __restrict__ in, W* __restrict__ out) {
    typedef typename VecOf<W, VW>::T V;
    constexpr int TA = 16 * VW * MA;
    constexpr int TB = 16 * VW * MB;
    constexpr int CPR = TB / VW;                 // chunks per smem row (power of two)
    constexpr int CHUNKS = TA * CPR / 256;       // chunks each thread stores
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* const sm = reinterpret_cast<V*>(smem_raw);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int ta = tid & 15;                     // micro-tile column along A
    const int tbg = tid >> 4;                    // micro-tile row group along B

    const I nTiles = (I)p.nTiles;
    I t = (I)blockIdx.x;
    if (t >= nTiles) return;
    const I stride = (I)gridDim.x;
    const I sInB = (I)p.sInB;
    const I sOutA = (I)p.sOutA;

    // v[mb][ma][k][j]: element (a = (ta + 16 ma)*VW + j, b = (tbg + 16 mb)*VW + k)
    W v[MB][MA][VW][VW];
    auto load = [&](const TileBase<I>& tb) {
        const int limA = (tb.mask & (1u << 14)) ? p.splitTail[0] : TA;
        const int limB = (tb.mask & (1u << 15)) ? p.splitTail[1] : TB;
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int b0 = (tbg + 16 * mb) * VW;
#pragma unroll
            for (int k = 0; k < VW; ++k) {
#pragma unroll
                for (int ma = 0; ma < MA; ++ma) {
                    const int a0 = (ta + 16 * ma) * VW;
                    if (a0 < limA && b0 < limB) {
                        const V x = __ldg(reinterpret_cast<const V*>(in + (tb.in + (I)(b0 + k) * sInB + a0)));
                        *reinterpret_cast<V*>(&v[mb][ma][k][0]) = x;
                    }
                }
            }
        }
    };

    TileBase<I> cur = decode_tile<I>(p, t, lane);
    load(cur);
    int buf = 0;
    for (; t < nTiles; t += stride) {
        V* const sb = sm + buf * (TA * CPR);
        // register transpose + swizzled staging: output row a = (ta + 16 ma)*VW + j
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
#pragma unroll
            for (int ma = 0; ma < MA; ++ma) {
#pragma unroll
                for (int j = 0; j < VW; ++j) {
                    W w[VW];
#pragma unroll
                    for (int k = 0; k < VW; ++k) w[k] = v[mb][ma][k][j];
                    const int a = (ta + 16 * ma) * VW + j;
                    const int c = (tbg + 16 * mb) ^ ((ta + 16 * ma) & (CPR - 1));
                    sb[a * CPR + c] = *reinterpret_cast<const V*>(w);
                }
            }
        }
        __syncthreads();
        const TileBase<I> now = cur;
        const I tn = t + stride;
        if (tn < nTiles) {
            cur = decode_tile<I>(p, tn, lane);
            load(cur);
        }
        const int limA = (now.mask & (1u << 14)) ? p.splitTail[0] : TA;
        const int limB = (now.mask & (1u << 15)) ? p.splitTail[1] : TB;
#pragma unroll
        for (int u = 0; u < CHUNKS; ++u) {
            const int q = tid + 256 * u;
            const int a = q / CPR;
            const int c = q % CPR;
            if (a < limA && c * VW < limB) {
                const V x = sb[a * CPR + (c ^ ((a / VW) & (CPR - 1)))];
                *reinterpret_cast<V*>(out + (now.out + (I)a * sOutA + c * VW)) = x;
            }
        }
        buf ^= 1;
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
template <typename W, int NREG, typename I>
static const void* tile_fn() {
    return reinterpret_cast<const void*>(&tile_kernel<W, NREG, I>);
}

static const void* pick_tile(int esize, int nreg, bool idx64) {
#define TT_PICK(W, I)                               \
    switch (nreg) {                                 \
        case 1: return tile_fn<W, 1, I>();          \
        case 2: return tile_fn<W, 2, I>();          \
        case 4: return tile_fn<W, 4, I>();          \
        case 8: return tile_fn<W, 8, I>();          \
        default: return nullptr;                    \
    }
    if (esize == 4) {
        if (idx64) { TT_PICK(uint32_t, int64_t) } else { TT_PICK(uint32_t, int32_t) }
    } else {
        if (idx64) { TT_PICK(uint64_t, int64_t) } else { TT_PICK(uint64_t, int32_t) }
    }
#undef TT_PICK
}

// 2-D kernel instantiations: (word, VW, MA, MB).  Tile TA x TB = 16*VW*MA x 16*VW*MB.
template <typename W, int VW, int MA, int MB>
static const void* t2d_fn(bool idx64) {
    return idx64 ? (const void*)&tiled2d_kernel<W, VW, MA, MB, int64_t>
                 : (const void*)&tiled2d_kernel<W, VW, MA, MB, int32_t>;
}

static const void* pick_tiled2d(int esize, int vec, int ta, int tb, bool idx64) {
    if (esize == 4 && vec == 4) {
        if (ta == 64 && tb == 64) return t2d_fn<uint32_t, 4, 1, 1>(idx64);
        if (ta == 128 && tb == 64) return t2d_fn<uint32_t, 4, 2, 1>(idx64);
        if (ta == 64 && tb == 128) return t2d_fn<uint32_t, 4, 1, 2>(idx64);
        if (ta == 128 && tb == 128) return t2d_fn<uint32_t, 4, 2, 2>(idx64);
    } else if (esize == 4 && vec == 2) {
        if (ta == 32 && tb == 64) return t2d_fn<uint32_t, 2, 1, 2>(idx64);
        if (ta == 64 && tb == 64) return t2d_fn<uint32_t, 2, 2, 2>(idx64);
    } else if (esize == 8 && vec == 2) {
        if (ta == 32 && tb == 32) return t2d_fn<uint64_t, 2, 1, 1>(idx64);
        if (ta == 64 && tb == 32) return t2d_fn<uint64_t, 2, 2, 1>(idx64);
        if (ta == 32 && tb == 64) return t2d_fn<uint64_t, 2, 1, 2>(idx64);
        if (ta == 64 && tb == 64) return t2d_fn<uint64_t, 2, 2, 2>(idx64);
    }
    return nullptr;
}

int cuda_occupancy(const OccQuery& q, const DeviceInfo& dev) {
    const void* fn = q.kernel == TT_KERNEL_TILE      ? pick_tile(q.esize, q.nreg, q.idx64)
                     : q.kernel == TT_KERNEL_TILED2D ? pick_tiled2d(q.esize, q.vec, q.ta, q.tb, q.idx64)
                                                     : nullptr;
    if (!fn) return 0;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dev.max_smem_per_block) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, q.threads, q.smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return blocks;
}

int launch_plan(const Plan& plan, const void* in, void* out, void* stream_) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const KernelChoice& kc = plan.kc;
    const int E = plan.prob.esize;
    if (kc.kernel == TT_KERNEL_COPY) {
        const int64_t n = plan.prob.vol;
        const int vec16 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
        if (E == 4)
            copy_kernel<uint32_t><<<kc.grid, kc.threads, 0, stream>>>(
                static_cast<const uint32_t*>(in), static_cast<uint32_t*>(out), n, vec16);
        else
            copy_kernel<uint64_t><<<kc.grid, kc.threads, 0, stream>>>(
                static_cast<const uint64_t*>(in), static_cast<uint64_t*>(out), n, vec16);
        return (int)cudaGetLastError();
    }
    if (kc.kernel == TT_KERNEL_TILE || kc.kernel == TT_KERNEL_TILED2D) {
        bool t2 = kc.kernel == TT_KERNEL_TILED2D;
        int threads = kc.threads, grid = kc.grid, smem = kc.smem;
        if (t2 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) &
                   (uintptr_t)(kc.vec * E - 1)) != 0) {
            // pointers not aligned to the vector width: generic tile fallback
            t2 = false;
            threads = kc.fb_threads;
            grid = kc.fb_grid;
            smem = kc.fb_smem;
        }
        const void* fn = t2 ? pick_tiled2d(E, kc.vec, kc.tile0, kc.tile1, kc.idx64)
                            : pick_tile(E, kc.nreg, kc.idx64);
        if (!fn) return (int)cudaErrorInvalidConfiguration;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return (int)e;
        }
        const void* pp = t2 ? (const void*)&plan.t2d : (const void*)&plan.tile;
        void* args[] = {const_cast<void*>(pp), (void*)&in, (void*)&out};
        return (int)cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, stream);
    }
    return (int)cudaErrorInvalidConfiguration;
}

}  // namespace tt
