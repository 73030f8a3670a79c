// kernels_sd.cu -- generic staged tile, slot-dim thread map (register pipeline
// and cp.async ring).
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#include "kern_common.cuh"
#include "kern_pick.h"

namespace tt {

template <typename W, int QM, int RM>
__global__ void __launch_bounds__(sizeof(W) >= 8 ? 384 : 512, 2)
tile_sd_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * (uint32_t)sizeof(W);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;

    uint32_t gin[QM], gout[QM], smp[QM], cntL[QM], cntS[QM];
#pragma unroll
    for (int q = 0; q < QM; ++q) smp[q] = 0;
    build_sd_phase<W, QM, RM>(p, 0, tid, NT, gin, smp, cntL);
    build_sd_phase<W, QM, RM>(p, 1, tid, NT, gout, smp, cntS);
    const int QL = p.sdQ[0], QS = p.sdQ[1];
    // uniform per-slot strides: global (elements) and staging (bytes)
    const uint32_t sIn = (uint32_t)p.tSin[p.sdSlot[0]];
    const uint32_t sOut = (uint32_t)p.tSout[p.sdSlot[1]];
    const uint32_t mIn = (uint32_t)p.tSm[p.sdSlot[0]] * (uint32_t)sizeof(W);
    const uint32_t mOut = (uint32_t)p.tSm[p.sdSlot[1]] * (uint32_t)sizeof(W);

    const uint32_t nTiles = (uint32_t)p.nTiles;
    const uint32_t G = (uint32_t)gridDim.x;
    const uint32_t t0 = (uint32_t)blockIdx.x;
    if (t0 >= nTiles) return;
    const uint32_t nIt = (nTiles - t0 + G - 1) / G;  // tiles t0 + it*G
    uint4* const ring = reinterpret_cast<uint4*>(smem_raw + p.ringOff);
    if ((tid >> 5) == 0)
        for (uint32_t it = (uint32_t)lane; it < 64u && it < nIt; it += 32) ring[it] = tile_entry(p, t0 + it * G);
    __syncthreads();
    auto base = [&](uint32_t it) {
        const uint4 e = ring[it & 63u];
        TileBase<uint32_t> b;
        b.in = e.x;
        b.out = e.y;
        b.need = e.z & 3u;
        return b;
    };

    W v[QM][RM];
    auto load = [&](const TileBase<uint32_t>& tb) {
        const uint32_t sh = 8u * tb.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QL) break;
            const uint32_t c = (cntL[q] >> sh) & 0xffu;
            // slot addresses chained (one IMAD.WIDE per slot)
            const W* __restrict__ src = opaque(in + tb.in + gin[q]);
            if (c == (uint32_t)RM) {
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    v[q][r] = ldg_(src);
                    src = elem_addr(src, sIn);
                }
            } else {
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    if ((uint32_t)r < c) v[q][r] = ldg_(src);
                    src = elem_addr(src, sIn);
                }
            }
        }
    };
    TileBase<uint32_t> cur = base(0);
    load(cur);

    uint32_t sb = sm0;
    for (uint32_t it = 0; it < nIt; ++it) {
        // stage the tile (input-side map)
        {
            const uint32_t sh = 8u * cur.need;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                if (q >= QL) break;
                const uint32_t c = (cntL[q] >> sh) & 0xffu;
                uint32_t a = sb + (smp[q] & 0xffffu);
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    if ((uint32_t)r < c) sts(a, v[q][r]);
                    a += mIn;
                }
            }
        }
        __syncthreads();
        if ((it & 31u) == 0 && it >= 32u && (tid >> 5) == 0) {  // bases of tiles it+32 .. it+63
            const uint32_t j = it + 32u + (uint32_t)lane;
            if (j < nIt) ring[j & 63u] = tile_entry(p, t0 + j * G);
        }
        const TileBase<uint32_t> now = cur;
        if (it + 1 < nIt) {
            cur = base(it + 1);
            load(cur);
        }
        // transposed read of the staged tile, coalesced writes (output-side map)
        {
            const uint32_t sh = 8u * now.need;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                if (q >= QS) break;
                const uint32_t c = (cntS[q] >> sh) & 0xffu;
                W* __restrict__ dst = opaque(out + now.out + gout[q]);
                uint32_t a = sb + (smp[q] >> 16);
                if (c == (uint32_t)RM) {
#pragma unroll
                    for (int r = 0; r < RM; ++r) {
                        stg_(dst, lds<W>(a));
                        dst = elem_addr(dst, sOut);
                        a += mOut;
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < RM; ++r) {
                        if ((uint32_t)r < c) stg_(dst, lds<W>(a));
                        dst = elem_addr(dst, sOut);
                        a += mOut;
                    }
                }
            }
        }
        sb = (sb == sm0) ? sm0 + sbytes : sm0;
    }
}


// ---------------------------------------------------------------------------
// slot-dim map with a cp.async ring: same thread maps, tables and staging
// layout as tile_sd_kernel, but the load phase copies global -> staging with
// cp.async (no data registers), so S-1 tiles are in flight per CTA instead of
// one tile's worth of registers (the loads-in-flight limit of 4-byte gathers,
// profiles/worst_cases/README.md).  Interleaved schedule t0 + k*G as in
// tile_sd_kernel; stage k % S holds tile k of this CTA.
// ---------------------------------------------------------------------------
template <typename W, int QM, int RM, int S>
__global__ void __launch_bounds__(512, 2)
tile_sd_async_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * (uint32_t)sizeof(W);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;

    uint32_t gin[QM], gout[QM], smp[QM], cntL[QM], cntS[QM];
#pragma unroll
    for (int q = 0; q < QM; ++q) smp[q] = 0;
    build_sd_phase<W, QM, RM>(p, 0, tid, NT, gin, smp, cntL);
    build_sd_phase<W, QM, RM>(p, 1, tid, NT, gout, smp, cntS);
    const int QL = p.sdQ[0], QS = p.sdQ[1];
    const uint32_t sIn = (uint32_t)p.tSin[p.sdSlot[0]];
    const uint32_t sOut = (uint32_t)p.tSout[p.sdSlot[1]];
    const uint32_t mIn = (uint32_t)p.tSm[p.sdSlot[0]] * (uint32_t)sizeof(W);
    const uint32_t mOut = (uint32_t)p.tSm[p.sdSlot[1]] * (uint32_t)sizeof(W);

    const uint32_t nTiles = (uint32_t)p.nTiles;
    const uint32_t G = (uint32_t)gridDim.x;
    const uint32_t t0 = (uint32_t)blockIdx.x;
    if (t0 >= nTiles) return;
    const uint32_t nIt = (nTiles - t0 + G - 1) / G;  // tiles t0 + it*G
    uint4* const ring = reinterpret_cast<uint4*>(smem_raw + p.ringOff);
    if ((tid >> 5) == 0)
        for (uint32_t it = (uint32_t)lane; it < 64u && it < nIt; it += 32) ring[it] = tile_entry(p, t0 + it * G);
    __syncthreads();
    auto base = [&](uint32_t it) {
        const uint4 e = ring[it & 63u];
        TileBase<uint32_t> b;
        b.in = e.x;
        b.out = e.y;
        b.need = e.z & 3u;
        return b;
    };

    // load phase of iteration it into the staging buffer at byte address sb
    auto issue = [&](uint32_t it, uint32_t sb) {
        const TileBase<uint32_t> tb = base(it);
        const uint32_t sh = 8u * tb.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QL) break;
            const uint32_t c = (cntL[q] >> sh) & 0xffu;
            const W* src = in + tb.in + gin[q];
            uint32_t a = sb + (smp[q] & 0xffffu);
#pragma unroll
            for (int r = 0; r < RM; ++r) {
                if ((uint32_t)r < c) cp_async<sizeof(W)>(a, src);
                src = elem_addr(src, sIn);
                a += mIn;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        if ((uint32_t)s < nIt) issue((uint32_t)s, sm0 + (uint32_t)s * sbytes);
        cp_async_commit();
    }
    uint32_t k = 0;
    for (uint32_t it = 0; it < nIt; ++it) {
        cp_async_wait<S - 2>();
        __syncthreads();
        if ((it & 31u) == 0 && it >= 32u && (tid >> 5) == 0) {  // bases of tiles it+32 .. it+63
            const uint32_t j = it + 32u + (uint32_t)lane;
            if (j < nIt) ring[j & 63u] = tile_entry(p, t0 + j * G);
        }
        // refill the stage read in the previous iteration (all threads are
        // past its reads: they passed this iteration's barrier)
        {
            const uint32_t itn = it + (uint32_t)(S - 1);
            const uint32_t kn = (k + S - 1) % S;
            if (itn < nIt) issue(itn, sm0 + kn * sbytes);
            cp_async_commit();
        }
        const TileBase<uint32_t> now = base(it);
        const uint32_t sb = sm0 + k * sbytes;
        const uint32_t sh = 8u * now.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QS) break;
            const uint32_t c = (cntS[q] >> sh) & 0xffu;
            W* __restrict__ dst = opaque(out + now.out + gout[q]);
            uint32_t a = sb + (smp[q] >> 16);
            if (c == (uint32_t)RM) {
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    stg_(dst, lds<W>(a));
                    dst = elem_addr(dst, sOut);
                    a += mOut;
                }
            } else {
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    if ((uint32_t)r < c) stg_(dst, lds<W>(a));
                    dst = elem_addr(dst, sOut);
                    a += mOut;
                }
            }
        }
        k = (k + 1 == (uint32_t)S) ? 0u : k + 1;
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
// slot-dim variant: (passes, slots) in {(1,16), (2,8), (4,4)}, 4/8-byte words,
// 32-bit indices
const void* pick_tile_sd(int esize, int q, int r, int stages) {
#define TT_PICKSD(W)                                                                  \
    if (stages == 3) {                                                                \
        if (q == 1 && r == 16) return (const void*)&tile_sd_async_kernel<W, 1, 16, 3>; \
        if (q == 2 && r == 8) return (const void*)&tile_sd_async_kernel<W, 2, 8, 3>;   \
        if (q == 4 && r == 4) return (const void*)&tile_sd_async_kernel<W, 4, 4, 3>;   \
        return nullptr;                                                               \
    }                                                                                 \
    if (stages == 4) {                                                                \
        if (q == 1 && r == 16) return (const void*)&tile_sd_async_kernel<W, 1, 16, 4>; \
        if (q == 2 && r == 8) return (const void*)&tile_sd_async_kernel<W, 2, 8, 4>;   \
        if (q == 4 && r == 4) return (const void*)&tile_sd_async_kernel<W, 4, 4, 4>;   \
        return nullptr;                                                               \
    }                                                                                 \
    if (q == 1 && r == 16) return (const void*)&tile_sd_kernel<W, 1, 16>;           \
    if (q == 2 && r == 8) return (const void*)&tile_sd_kernel<W, 2, 8>;             \
    if (q == 4 && r == 4) return (const void*)&tile_sd_kernel<W, 4, 4>;             \
    return nullptr;
    if (esize == 4) { TT_PICKSD(uint32_t) }
    if (esize == 8) { TT_PICKSD(uint64_t) }
    return nullptr;
#undef TT_PICKSD
}

}  // namespace tt
