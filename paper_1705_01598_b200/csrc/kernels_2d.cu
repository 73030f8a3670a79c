// kernels_2d.cu -- copy, row copy (TiledCopy) and the 2-D tiled
// transposes (Tiled): vectorised, scalar, scalar with a cp.async ring.
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#include "kern_common.cuh"
#include "kern_pick.h"

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

// Output row r (r over output dims 1..n-1 in output order) is out[r*L, r*L+L)
// and the contiguous input row at base(r) = sum_j x_j * S_in_j.  Each warp
// copies a contiguous range of rows: the first base is decoded with
// Algorithm 1 (lane j holds digit x_j), the next ones by a lane-parallel
// odometer step (ballot finds the first digit that does not wrap).
template <typename W, typename I>
__global__ void __launch_bounds__(256)
rowcopy_kernel(const __grid_constant__ RowParams p, const W* __restrict__ in, W* __restrict__ out) {
    // 4-byte words: 16 loads in flight per lane (U = 4 left rows of odd
    // length at 0.67 of memcpy on B200); 8/16-byte words: 4 (8 measured
    // 1-4 % slower)
    constexpr int U = sizeof(W) == 4 ? 16 : 4;
    const int lane = threadIdx.x & 31;
    const I nWarps = (I)(((uint64_t)gridDim.x * blockDim.x) >> 5);
    const I warp = (I)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const I nRows = (I)p.nRows;
    const I per = (nRows + nWarps - 1) / nWarps;
    const I r0 = warp * per;
    if (r0 >= nRows) return;
    const I r1 = min(r0 + per, nRows);
    // segmented rows: lane 0's digit is the segment index (planner.cpp)
    const bool segd = p.nseg > 1;
    const I nseg = (I)p.nseg, seg = (I)p.seg, segTail = (I)p.segTail, rowFull = (I)p.rowFull;
    I obase = segd ? (r0 / nseg) * rowFull + (r0 % nseg) * seg : r0 * rowFull;

    I x = 0, d = 1, s = 0;
    if (lane < p.h) {
        d = (I)p.rD[lane];
        s = (I)p.rSin[lane];
        if constexpr (sizeof(I) == 4) {
            const uint32_t q1 = fast_div((uint32_t)r0, p.gMC[lane], p.gLC[lane]);
            x = (I)(q1 - fast_div(q1, p.gMD[lane], p.gLD[lane]) * (uint32_t)d);
        } else {
            x = (r0 / (I)p.rC[lane]) % d;
        }
    }
    I base = warp_sum<I>(x * s);
    // odometer step to the next row: returns the input base delta
    auto step = [&]() {
        const uint32_t wraps = __ballot_sync(0xffffffffu, lane < p.h && x == d - 1);
        const int f = __ffs(~wraps) - 1;
        I delta = 0;
        if (lane < f) { delta = (I)0 - (d - 1) * s; x = 0; }
        else if (lane == f) { delta = s; x += 1; }
        return warp_sum<I>(delta);
    };
    if (!segd && (I)p.seg <= (I)(32 * U)) {
        // short rows (one load per lane and word slot per row): the next
        // row's loads are issued before this row's stores, so two rows per
        // warp are in flight instead of one (rows of 0.7-1 KB were
        // latency-bound at ~0.77-0.88 of memcpy)
        const I L = (I)p.seg;
        W t[U], t2[U];
        {
            const W* __restrict__ src = opaque(in + base);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (lane + 32 * u < L) t[u] = ldg_(src + lane + 32 * u);
        }
        for (I r = r0; r < r1; ++r) {
            base += step();
            if (r + 1 < r1) {
                const W* __restrict__ src = opaque(in + base);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (lane + 32 * u < L) t2[u] = ldg_(src + lane + 32 * u);
            }
            W* __restrict__ dst = opaque(out + obase);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (lane + 32 * u < L) stg_(dst + lane + 32 * u, t[u]);
            obase += L;
#pragma unroll
            for (int u = 0; u < U; ++u) t[u] = t2[u];
        }
        return;
    }
    for (I r = r0; r < r1; ++r) {
        const W* __restrict__ src = opaque(in + base);
        W* __restrict__ dst = opaque(out + obase);
        const I segIdx = segd ? __shfl_sync(0xffffffffu, x, 0) : (I)0;
        const I L = (segd && segIdx == nseg - 1) ? segTail : seg;
        for (I c = lane; c < L; c += 32 * U) {
            W t[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c + 32 * u < L) t[u] = ldg_(src + c + 32 * u);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c + 32 * u < L) stg_(dst + c + 32 * u, t[u]);
        }
        base += step();  // odometer step to row r+1
        // output rows are dense in output order: the next segment, or the
        // next row's first segment (after this row's last, segTail long)
        obase += L;
    }
}



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
        const int limA = (tb.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (tb.need & 2u) ? p.splitTail[1] : TB;
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
        const int limA = (now.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (now.need & 2u) ? p.splitTail[1] : TB;
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
// scalar 2-D tiled transpose: the Tiled class when the two
// fastest dims do not allow vectors (odd extents).  256 threads = 32 lanes
// along A x 8 along B; each thread moves MA x MB elements of a TA = 32*MA by
// TB = 8*MB tile through shared memory rows of TB+1 elements -- the paper's
// L x (L+1) padding, conflict-free for both the staging store
// (lanes along A) and the transposed read (lanes along B).
// ---------------------------------------------------------------------------
template <typename W, int MA, int MB, typename I>
__global__ void __launch_bounds__(256)
tiled2d_s_kernel(const __grid_constant__ Tiled2DParams p, const W* __restrict__ in, W* __restrict__ out) {
    constexpr int TA = 32 * MA;
    constexpr int TB = 8 * MB;
    constexpr int RS = TB + 1;                       // padded row stride (elements)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    constexpr uint32_t BUF = (uint32_t)(TA * RS * sizeof(W));
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int wid = tid >> 5;                        // 8 warps

    const I nTiles = (I)p.nTiles;
    I t = (I)blockIdx.x;
    if (t >= nTiles) return;
    const I stride = (I)gridDim.x;
    const I sInB = (I)p.sInB;
    const I sOutA = (I)p.sOutA;

    W v[MB][MA];  // element (a = lane + 32 ma, b = wid + 8 mb)
    auto load = [&](const TileBase<I>& tb) {
        const int limA = (tb.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (tb.need & 2u) ? p.splitTail[1] : TB;
        const W* __restrict__ src = opaque(in + tb.in);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int b = wid + 8 * mb;
#pragma unroll
            for (int ma = 0; ma < MA; ++ma) {
                const int a = lane + 32 * ma;
                if (a < limA && b < limB) v[mb][ma] = ldg_(src + ((I)b * sInB + a));
            }
        }
    };
    TileBase<I> cur = decode_tile<I>(p, t, lane);
    load(cur);
    uint32_t sb = sm0;
    for (; t < nTiles; t += stride) {
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int ma = 0; ma < MA; ++ma)
                sts(sb + (uint32_t)(((lane + 32 * ma) * RS + wid + 8 * mb) * sizeof(W)), v[mb][ma]);
        __syncthreads();
        const TileBase<I> now = cur;
        const I tn = t + stride;
        if (tn < nTiles) {
            cur = decode_tile<I>(p, tn, lane);
            load(cur);
        }
        const int limA = (now.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (now.need & 2u) ? p.splitTail[1] : TB;
        W* __restrict__ dst = opaque(out + now.out);
        // output row a = wid + 8 j, elements b = lane + 32 u
#pragma unroll
        for (int j = 0; j < TA / 8; ++j) {
            const int a = wid + 8 * j;
#pragma unroll
            for (int u = 0; u < TB / 32; ++u) {
                const int b = lane + 32 * u;
                if (a < limA && b < limB)
                    stg_(dst + ((I)a * sOutA + b), lds<W>(sb + (uint32_t)((a * RS + b) * sizeof(W))));
            }
        }
        sb = (sb == sm0) ? sm0 + BUF : sm0;
    }
}

// scalar 2-D tile, asynchronous-copy pipeline: the same tiles, thread map
// and padded staging rows as tiled2d_s_kernel, but the loads go straight to
// shared memory with cp.async (no data registers), so S-1 tiles per CTA are
// in flight instead of one (ncu on odd-extent fp64 cases of the register
// version: 24 warps/SM, long-scoreboard 46 %, DRAM traffic = algorithmic --
// latency-bound, not traffic-bound).
template <typename W, int MA, int MB, typename I, int S>
__global__ void __launch_bounds__(256)
tiled2d_sa_kernel(const __grid_constant__ Tiled2DParams p, const W* __restrict__ in, W* __restrict__ out) {
    constexpr int TA = 32 * MA;
    constexpr int TB = 8 * MB;
    constexpr int RS = TB + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    constexpr uint32_t BUF = (uint32_t)(TA * RS * sizeof(W));
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int wid = tid >> 5;

    const I nTiles = (I)p.nTiles;
    I t = (I)blockIdx.x;
    if (t >= nTiles) return;
    const I stride = (I)gridDim.x;
    const I sInB = (I)p.sInB;
    const I sOutA = (I)p.sOutA;

    auto issue = [&](const TileBase<I>& tb, uint32_t sb) {
        const int limA = (tb.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (tb.need & 2u) ? p.splitTail[1] : TB;
        const W* __restrict__ src = opaque(in + tb.in);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const int b = wid + 8 * mb;
#pragma unroll
            for (int ma = 0; ma < MA; ++ma) {
                const int a = lane + 32 * ma;
                if (a < limA && b < limB)
                    cp_async<sizeof(W)>(sb + (uint32_t)((a * RS + b) * sizeof(W)), src + ((I)b * sInB + a));
            }
        }
    };
    TileBase<I> q[S - 1];
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        const I tj = t + (I)j * stride;
        if (tj < nTiles) {
            q[j] = decode_tile<I>(p, tj, lane);
            issue(q[j], sm0 + (uint32_t)j * BUF);
        }
        cp_async_commit();
    }
    int stage = 0;
    for (; t < nTiles; t += stride) {
        cp_async_wait<S - 2>();  // this thread's copies for tile t have landed
        __syncthreads();         // ... and everyone's; last iteration's stage is free
        const I tn = t + (I)(S - 1) * stride;
        const bool more = tn < nTiles;
        TileBase<I> nw;
        if (more) {
            nw = decode_tile<I>(p, tn, lane);
            issue(nw, sm0 + (uint32_t)((stage + S - 1) % S) * BUF);
        }
        cp_async_commit();
        const TileBase<I> now = q[0];
        const uint32_t sb = sm0 + (uint32_t)stage * BUF;
        const int limA = (now.need & 1u) ? p.splitTail[0] : TA;
        const int limB = (now.need & 2u) ? p.splitTail[1] : TB;
        W* __restrict__ dst = opaque(out + now.out);
#pragma unroll
        for (int j = 0; j < TA / 8; ++j) {
            const int a = wid + 8 * j;
#pragma unroll
            for (int u = 0; u < TB / 32; ++u) {
                const int b = lane + 32 * u;
                if (a < limA && b < limB)
                    stg_(dst + ((I)a * sOutA + b), lds<W>(sb + (uint32_t)((a * RS + b) * sizeof(W))));
            }
        }
#pragma unroll
        for (int j = 0; j + 1 < S - 1; ++j) q[j] = q[j + 1];
        if (more) q[S - 2] = nw;
        stage = (stage + 1 == S) ? 0 : stage + 1;
    }
    cp_async_wait<0>();
}

const void* pick_rowcopy(int esize, bool idx64) {
    switch (esize) {
        case 4: return idx64 ? (const void*)&rowcopy_kernel<uint32_t, int64_t>
                             : (const void*)&rowcopy_kernel<uint32_t, uint32_t>;
        case 8: return idx64 ? (const void*)&rowcopy_kernel<uint64_t, int64_t>
                             : (const void*)&rowcopy_kernel<uint64_t, uint32_t>;
        case 16: return idx64 ? (const void*)&rowcopy_kernel<uint4, int64_t>
                              : (const void*)&rowcopy_kernel<uint4, uint32_t>;
        default: return nullptr;
    }
}

// 2-D kernel instantiations: (word, VW, MA, MB).  Tile TA x TB = 16*VW*MA x 16*VW*MB.
template <typename W, int VW, int MA, int MB>
static const void* t2d_fn(bool idx64) {
    return idx64 ? (const void*)&tiled2d_kernel<W, VW, MA, MB, int64_t>
                 : (const void*)&tiled2d_kernel<W, VW, MA, MB, uint32_t>;
}

template <typename W, int MA, int MB>
static const void* t2ds_fn(bool idx64) {
    return idx64 ? (const void*)&tiled2d_s_kernel<W, MA, MB, int64_t>
                 : (const void*)&tiled2d_s_kernel<W, MA, MB, uint32_t>;
}

template <typename W, int MA, int MB>
static const void* t2dsa_fn(int stages) {
    return stages == 4 ? (const void*)&tiled2d_sa_kernel<W, MA, MB, uint32_t, 4>
                       : (const void*)&tiled2d_sa_kernel<W, MA, MB, uint32_t, 3>;
}

// scalar 2-D kernel with the cp.async ring (3 or 4 stages, 32-bit indices)
const void* pick_tiled2d_async(int esize, int ta, int tb, int stages) {
    if (esize == 4 && ta == 64 && tb == 64) return t2dsa_fn<uint32_t, 2, 8>(stages);
    if (esize == 4 && ta == 128 && tb == 64) return t2dsa_fn<uint32_t, 4, 8>(stages);
    if (esize == 4 && ta == 64 && tb == 128) return t2dsa_fn<uint32_t, 2, 16>(stages);
    if (esize == 8 && ta == 64 && tb == 64) return t2dsa_fn<uint64_t, 2, 8>(stages);
    if (esize == 8 && ta == 32 && tb == 64) return t2dsa_fn<uint64_t, 1, 8>(stages);
    if (esize == 8 && ta == 64 && tb == 32) return t2dsa_fn<uint64_t, 2, 4>(stages);
    return nullptr;
}

const void* pick_tiled2d(int esize, int vec, int ta, int tb, bool idx64) {
    if (vec == 1) {  // scalar 2-D kernel: TA = 32*MA, TB = 8*MB
        if (esize == 4 && ta == 64 && tb == 64) return t2ds_fn<uint32_t, 2, 8>(idx64);
        if (esize == 4 && ta == 128 && tb == 64) return t2ds_fn<uint32_t, 4, 8>(idx64);
        if (esize == 4 && ta == 64 && tb == 128) return t2ds_fn<uint32_t, 2, 16>(idx64);
        if (esize == 8 && ta == 64 && tb == 64) return t2ds_fn<uint64_t, 2, 8>(idx64);
        if (esize == 8 && ta == 32 && tb == 64) return t2ds_fn<uint64_t, 1, 8>(idx64);
        if (esize == 8 && ta == 64 && tb == 32) return t2ds_fn<uint64_t, 2, 4>(idx64);
        return nullptr;
    }
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

const void* pick_copy() { return (const void*)&copy_kernel<uint32_t>; }

}  // namespace tt
