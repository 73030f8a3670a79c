// kernels_tile.cu -- generic staged tile (Tiled / Packed / PackedSplit classes,
// P:L121-161) with per-thread slot tables, register double buffer or cp.async ring.
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#include "kern_common.cuh"
#include "kern_pick.h"

namespace tt {

// Per slot r (tile element k = tid + r*NT): gin/gout = global minor offsets
// (Eqs. 4, 5), sin/sout = staging byte offsets of the load element and of the
// store element (Eq. 6 through the padded layout).  `flags` holds 4 bits per
// slot: (load elem inside ragged A-chunk, ... B-chunk, store elem inside
// ragged A-chunk, ... B-chunk); a slot is valid in a ragged tile iff its bits
// cover the tile's `need`.
template <typename W, int NREG, typename I, int ACC = 0>
__global__ void __launch_bounds__(NREG >= 16 ? 256 : 512,
                                  (NREG >= 16 ? 2 : (ACC || sizeof(I) == 8 || (NREG >= 8 && sizeof(W) >= 8) ? 1 : 2)))
tile_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * (uint32_t)sizeof(W);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;

    // Per-thread loop-invariant minor positions (Eqs. 4-6; the
    // register arrays of P:L155-159).
    I gin[NREG], gout[NREG];
    uint32_t spk[NREG];  // staging byte offsets: load element (low 16 bits), store element (high)
    typedef typename std::conditional<(NREG > 8), uint64_t, uint32_t>::type FlagT;
    FlagT flags = 0;
    const int nmine = (p.V > tid) ? min(NREG, (p.V - tid + NT - 1) / NT) : 0;
    const bool allSlots = p.V == NT * NREG;  // CTA-uniform
    build_slots<W, NREG, I, FlagT>(p, tid, NT, nmine, gin, gout, spk, flags);
    typedef typename std::conditional<(4 * NREG > 32), uint64_t, uint32_t>::type MaskT;
    MaskT lmask, smask;
    slot_masks<NREG>(flags, nmine, lmask, smask);

    // Tile schedule: a contiguous range per CTA walked with the odometer, or
    // (p.interleave) tiles blockIdx.x + k*gridDim.x so that concurrently
    // running CTAs work on neighbouring tiles, each found with Algorithm 1.
    const I nTiles = (I)p.nTiles;
    const I G = (I)gridDim.x;
    const bool il = p.interleave != 0;
    const I t0 = il ? (I)blockIdx.x : (I)(((uint64_t)nTiles * blockIdx.x) / G);
    const I t1 = il ? nTiles : (I)(((uint64_t)nTiles * (blockIdx.x + 1)) / G);
    const I step = il ? G : (I)1;
    if (t0 >= t1) return;
    // tile bases: 32-bit plans read them from a shared ring (tile_entry,
    // 32 tiles decoded at a time by one warp); 64-bit plans keep the
    // warp-parallel walker
    constexpr bool kRingBases = sizeof(I) == 4;
    const uint32_t nIt = (uint32_t)((t1 - t0 + step - 1) / step);
    uint4* const ring = reinterpret_cast<uint4*>(smem_raw + p.ringOff);
    if constexpr (kRingBases) {
        if ((tid >> 5) == 0)
            for (uint32_t it = (uint32_t)lane; it < 64u && it < nIt; it += 32)
                ring[it] = tile_entry(p, (uint32_t)t0 + it * (uint32_t)step);
        __syncthreads();
    }
    auto ring_base = [&](uint32_t it) {
        const uint4 e = ring[it & 63u];
        TileBase<I> b;
        b.in = (I)e.x;
        b.out = (I)e.y;
        b.need = e.z & 3u;
        return b;
    };
    GridWalker<I> walk(p, lane, !kRingBases);

    W v[NREG];
    auto load = [&](const TileBase<I>& tb) {
        const W* __restrict__ src = opaque(in + tb.in);
        if (tb.need == 0 && allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r) v[r] = ldg_(elem_addr(src, gin[r]));
        } else {
            const uint32_t m = (uint32_t)(lmask >> (tb.need * NREG));
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (m & (1u << r)) v[r] = ldg_(elem_addr(src, gin[r]));
        }
    };
    // accumulate plans: the old output values of a tile, prefetched one
    // iteration ahead (after the previous tile's writes) so the read of `out`
    // is not exposed in the store phase
    W ov[ACC ? NREG : 1];
    auto load_out = [&](const TileBase<I>& tb) {
        if constexpr (ACC != 0) {
            if (p.betaZero) return;
            const W* __restrict__ o = opaque(out + tb.out);
            const uint32_t m = (uint32_t)(smask >> (tb.need * NREG));
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (m & (1u << r)) ov[r] = ldgo_(elem_addr(o, gout[r]));
        }
    };
    TileBase<I> cur;
    if constexpr (kRingBases) cur = ring_base(0);
    else cur = walk.seek(t0);
    load(cur);
    load_out(cur);

    uint32_t sb = sm0;
    uint32_t it = 0;
    for (I t = t0; t < t1; t += step, ++it) {
        // stage the tile in input order
        if (allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r) sts(sb + (spk[r] & 0xffffu), v[r]);
        } else {
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (r < nmine) sts(sb + (spk[r] & 0xffffu), v[r]);
        }
        __syncthreads();
        if constexpr (kRingBases) {
            if ((it & 31u) == 0 && it >= 32u && (tid >> 5) == 0) {  // bases of tiles it+32 .. it+63
                const uint32_t j = it + 32u + (uint32_t)lane;
                if (j < nIt) ring[j & 63u] = tile_entry(p, (uint32_t)t0 + j * (uint32_t)step);
            }
        }
        // issue the next tile's global loads before writing this one
        const TileBase<I> now = cur;
        if (t + step < t1) {
            if constexpr (kRingBases) cur = ring_base(it + 1);
            else cur = il ? walk.seek(t + step) : walk.next(cur);
            load(cur);
        }
        // transposed read of shared memory (Eq. 6), coalesced writes (Eq. 5)
        W* __restrict__ dst = opaque(out + now.out);
        if (now.need == 0 && allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                put_out<W, ACC>(elem_addr(dst, gout[r]), lds<W>(sb + (spk[r] >> 16)),
                                ov[ACC ? r : 0], p);
        } else {
            const uint32_t m = (uint32_t)(smask >> (now.need * NREG));
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (m & (1u << r))
                    put_out<W, ACC>(elem_addr(dst, gout[r]), lds<W>(sb + (spk[r] >> 16)),
                                    ov[ACC ? r : 0], p);
        }
        if (t + step < t1) load_out(cur);
        // Two buffers: the next iteration writes the other buffer, whose
        // readers (previous tile) all passed this iteration's barrier.
        sb = (sb == sm0) ? sm0 + sbytes : sm0;
    }
}

template <typename W, int NREG, typename I, int S>
__global__ void __launch_bounds__(NREG >= 16 ? 256 : 512, 2)
tile_async_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * (uint32_t)sizeof(W);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;

    I gin[NREG], gout[NREG];
    uint32_t spk[NREG];
    typedef typename std::conditional<(NREG > 8), uint64_t, uint32_t>::type FlagT;
    FlagT flags = 0;
    const int nmine = (p.V > tid) ? min(NREG, (p.V - tid + NT - 1) / NT) : 0;
    const bool allSlots = p.V == NT * NREG;
    build_slots<W, NREG, I, FlagT>(p, tid, NT, nmine, gin, gout, spk, flags);

    const I nTiles = (I)p.nTiles;
    const I G = (I)gridDim.x;
    const I t0 = (I)(((uint64_t)nTiles * blockIdx.x) / G);
    const I t1 = (I)(((uint64_t)nTiles * (blockIdx.x + 1)) / G);
    if (t0 >= t1) return;
    GridWalker<I> walk(p, lane);

    auto issue = [&](const TileBase<I>& tb, uint32_t stage) {
        const W* __restrict__ src = opaque(in + tb.in);
        if (tb.need == 0 && allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                cp_async<sizeof(W)>(stage + (spk[r] & 0xffffu), elem_addr(src, gin[r]));
        } else {
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (r < nmine && ((flags >> (4 * r)) & tb.need) == tb.need)
                    cp_async<sizeof(W)>(stage + (spk[r] & 0xffffu), elem_addr(src, gin[r]));
        }
    };

    // prologue: tiles t0 .. t0+S-2 in flight
    TileBase<I> q[S - 1];  // q[0] = the tile written next
    TileBase<I> cur = walk.seek(t0);
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        if (t0 + j < t1) {
            if (j > 0) cur = walk.next(cur);
            q[j] = cur;
            issue(cur, sm0 + (uint32_t)j * sbytes);
        }
        cp_async_commit();
    }
    int stage = 0;  // stage of tile t
    for (I t = t0; t < t1; ++t) {
        cp_async_wait<S - 2>();  // this thread's copies for tile t have landed
        __syncthreads();         // ... and everyone's; the stage read last iteration is free
        TileBase<I> nw;
        const bool more = t + (S - 1) < t1;
        if (more) {
            cur = walk.next(cur);
            nw = cur;
            const int ns = (stage + S - 1) % S;
            issue(cur, sm0 + (uint32_t)ns * sbytes);
        }
        cp_async_commit();
        // transposed read of the staged tile (Eq. 6), coalesced writes (Eq. 5)
        const TileBase<I> now = q[0];
        const uint32_t sb = sm0 + (uint32_t)stage * sbytes;
        W* __restrict__ dst = opaque(out + now.out);
        if (now.need == 0 && allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r) stg_(elem_addr(dst, gout[r]), lds<W>(sb + (spk[r] >> 16)));
        } else {
            const uint32_t needOut = now.need << 2;
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (r < nmine && ((flags >> (4 * r)) & needOut) == needOut)
                    stg_(elem_addr(dst, gout[r]), lds<W>(sb + (spk[r] >> 16)));
        }
#pragma unroll
        for (int j = 0; j + 1 < S - 1; ++j) q[j] = q[j + 1];
        if (more) q[S - 2] = nw;
        stage = (stage + 1 == S) ? 0 : stage + 1;
    }
    cp_async_wait<0>();
}

template <typename W, int NREG, typename I>
static const void* tile_fn() {
    return reinterpret_cast<const void*>(&tile_kernel<W, NREG, I>);
}

// accumulate variant (f-3): 4/8-byte words, 32-bit indices
const void* pick_tile_acc(int esize, int nreg) {
#define TT_PICKACC(W)                                                               \
    switch (nreg) {                                                                 \
        case 1: return (const void*)&tile_kernel<W, 1, uint32_t, 1>;               \
        case 2: return (const void*)&tile_kernel<W, 2, uint32_t, 1>;               \
        case 4: return (const void*)&tile_kernel<W, 4, uint32_t, 1>;               \
        case 8: return (const void*)&tile_kernel<W, 8, uint32_t, 1>;               \
        default: return nullptr;                                                    \
    }
    if (esize == 4) { TT_PICKACC(uint32_t) }
    if (esize == 8) { TT_PICKACC(uint64_t) }
    return nullptr;
#undef TT_PICKACC
}

const void* pick_tile(int esize, int nreg, bool idx64) {
#define TT_PICK(W, I)                               \
    switch (nreg) {                                 \
        case 1: return tile_fn<W, 1, I>();          \
        case 2: return tile_fn<W, 2, I>();          \
        case 4: return tile_fn<W, 4, I>();          \
        case 8: return tile_fn<W, 8, I>();          \
        case 16: return tile_fn<W, 16, I>();        \
        default: return nullptr;                    \
    }
#define TT_PICK8(W, I)                              \
    switch (nreg) {                                 \
        case 1: return tile_fn<W, 1, I>();          \
        case 2: return tile_fn<W, 2, I>();          \
        case 4: return tile_fn<W, 4, I>();          \
        case 8: return tile_fn<W, 8, I>();          \
        default: return nullptr;                    \
    }
    // 16 slots only with 32-bit indices (the planner never pairs them with
    // 64-bit indices: 256-thread CTAs could not hold the tables)
    if (idx64 && nreg > 8) return nullptr;
    if (esize == 4) {
        if (idx64) { TT_PICK8(uint32_t, int64_t) } else { TT_PICK(uint32_t, uint32_t) }
    } else if (esize == 8) {
        if (idx64) { TT_PICK8(uint64_t, int64_t) } else { TT_PICK(uint64_t, uint32_t) }
    } else if (esize == 16) {  // widened words: at most 4 slots (register budget)
        switch (nreg) {
            case 1: return idx64 ? tile_fn<uint4, 1, int64_t>() : tile_fn<uint4, 1, uint32_t>();
            case 2: return idx64 ? tile_fn<uint4, 2, int64_t>() : tile_fn<uint4, 2, uint32_t>();
            case 4: return idx64 ? tile_fn<uint4, 4, int64_t>() : tile_fn<uint4, 4, uint32_t>();
            default: return nullptr;
        }
    }
    return nullptr;
#undef TT_PICK8
#undef TT_PICK
}

// asynchronous-copy tile: 3 stages, 32-bit indices, 4/8/16-byte words
const void* pick_tile_async(int esize, int nreg, bool idx64) {
    if (idx64) return nullptr;
#define TT_PICKA(W)                                                                  \
    switch (nreg) {                                                                  \
        case 1: return (const void*)&tile_async_kernel<W, 1, uint32_t, 3>;           \
        case 2: return (const void*)&tile_async_kernel<W, 2, uint32_t, 3>;           \
        case 4: return (const void*)&tile_async_kernel<W, 4, uint32_t, 3>;           \
        case 8: return (const void*)&tile_async_kernel<W, 8, uint32_t, 3>;           \
        case 16: return (const void*)&tile_async_kernel<W, 16, uint32_t, 3>;         \
        default: return nullptr;                                                     \
    }
    if (esize == 4) { TT_PICKA(uint32_t) }
    if (esize == 8) { TT_PICKA(uint64_t) }
    if (esize == 16 && nreg <= 4) { TT_PICKA(uint4) }
    return nullptr;
#undef TT_PICKA
}

}  // namespace tt
