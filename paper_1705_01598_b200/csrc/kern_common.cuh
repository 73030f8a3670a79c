// kern_common.cuh -- device helpers shared by the kernel translation units
// (kernels_*.cu): shared/global access wrappers, the Algorithm-1 tile decode
// and warp-parallel grid walker, the generic tile's per-slot
// tables (Eqs. 4-6), cp.async wrappers.
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "tt_internal.h"

namespace tt {

// ---------------------------------------------------------------------------
// shared memory by 32-bit shared-window byte address (no generic->shared
// conversions in the hot loop)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts(uint32_t a, uint64_t v) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ void sts(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
template <typename W> __device__ __forceinline__ W lds(uint32_t a);
template <> __device__ __forceinline__ uint32_t lds<uint32_t>(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ uint64_t lds<uint64_t>(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ uint4 lds<uint4>(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 ldg_(const uint4* p) { return __ldg(p); }
// Global stores through explicit st.global: pointers built by elem_addr (a
// mad.wide in inline PTX) are generic to the compiler, which would otherwise
// emit generic ST instead of STG.
__device__ __forceinline__ void stg_(uint32_t* p, uint32_t v) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void stg_(uint64_t* p, uint64_t v) {
    asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void stg_(uint4* p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint32_t ldgo_(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ldgo_(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ldgo_(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg_(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t ldg_(const uint64_t* p) {
    return __ldg(reinterpret_cast<const unsigned long long*>(p));
}

// Hide a per-tile base pointer from the optimiser so that `base + offset`
// stays one IMAD.WIDE.U32 per access instead of a re-associated 64-bit add.
template <typename T>
__device__ __forceinline__ T* opaque(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}

// base + off elements as one mad.wide.u32 (32-bit offsets stay 32-bit in
// registers instead of being hoisted as 64-bit byte offsets).
template <typename W>
__device__ __forceinline__ const W* elem_addr(const W* base, uint32_t off) {
    const W* r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(off), "n"((int)sizeof(W)), "l"(base));
    return r;
}
template <typename W>
__device__ __forceinline__ W* elem_addr(W* base, uint32_t off) {
    W* r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(off), "n"((int)sizeof(W)), "l"(base));
    return r;
}
template <typename W>
__device__ __forceinline__ const W* elem_addr(const W* base, int64_t off) { return base + off; }
template <typename W>
__device__ __forceinline__ W* elem_addr(W* base, int64_t off) { return base + off; }

// ---------------------------------------------------------------------------
// generic staged tile
// ---------------------------------------------------------------------------
template <typename I>
struct TileBase {
    I in, out;
    uint32_t need;   // bit 0: ragged last chunk of split dim A, bit 1: of split dim B
};

// n / d for n < 2^31 with the planner's magic (m, l): (umulhi(n, m) + n) >> l.
__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t m, uint32_t l) {
    return (__umulhi(n, m) + n) >> l;
}

// Warp-parallel walk over the tile grid (the "major" dims M̄_mk).
// Lane i < h owns grid dim i: its extent, its input/output strides and its
// digit of the current tile index, all in registers (indexing the kernel
// parameters per lane would serialise the constant cache).
//  * seek(t): Algorithm 1 -- every lane evaluates its term
//    mod(floor(t / c_i), d_i) * stride_i (multiply-shift division for 32-bit
//    indices) and an XOR butterfly sums the terms for Eq. (2) and Eq. (3) in
//    ONE common order (R3).
//  * next(): the tile t+1 from tile t without any division: a ballot finds the
//    first digit that does not wrap; its lane's precomputed carry (its stride
//    minus the wrapped lower digits' spans, an exclusive warp scan done once)
//    is broadcast with one shuffle per side.
// Split dims report their ragged last chunk (PackedSplit edge).
template <typename I>
struct GridWalker {
    I d, x, sIn, sOut, cIn, cOut;
    uint32_t mC, lC, mD, lD;
    I cC;
    uint32_t splitBit;  // 1 / 2 if this lane is split dim A / B with a ragged tail
    int h, lane;

    template <typename P>
    __device__ __forceinline__ GridWalker(const P& p, int lane_, bool enabled = true) : lane(lane_) {
        h = enabled ? p.h : 0;
        d = 1; sIn = 0; sOut = 0; x = 0; cC = 1;
        mC = 1; lC = 0; mD = 1; lD = 0;
        splitBit = 0;
        if (lane < h) {
            d = (I)p.gD[lane];
            sIn = (I)p.gSin[lane];
            sOut = (I)p.gSout[lane];
            cC = (I)p.gC[lane];
            mC = p.gMC[lane]; lC = p.gLC[lane]; mD = p.gMD[lane]; lD = p.gLD[lane];
            if (p.nSplit > 0 && lane == p.splitLane[0] && p.splitTail[0] != p.splitChunk[0]) splitBit |= 1u;
            if (p.nSplit > 1 && lane == p.splitLane[1] && p.splitTail[1] != p.splitChunk[1]) splitBit |= 2u;
        }
        // exclusive scan of the wrapped spans (d_i - 1) * stride_i over lanes
        I spanIn = (lane < h) ? (d - 1) * sIn : (I)0;
        I spanOut = (lane < h) ? (d - 1) * sOut : (I)0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const I ui = __shfl_up_sync(0xffffffffu, spanIn, o);
            const I uo = __shfl_up_sync(0xffffffffu, spanOut, o);
            if (lane >= o) { spanIn += ui; spanOut += uo; }
        }
        const I exIn = __shfl_up_sync(0xffffffffu, spanIn, 1);
        const I exOut = __shfl_up_sync(0xffffffffu, spanOut, 1);
        cIn = sIn - (lane > 0 ? exIn : (I)0);
        cOut = sOut - (lane > 0 ? exOut : (I)0);
    }

    __device__ __forceinline__ uint32_t need() const {
        const bool last = lane < h && x == d - 1;
        const uint32_t a = __ballot_sync(0xffffffffu, last && (splitBit & 1u));
        const uint32_t b = __ballot_sync(0xffffffffu, last && (splitBit & 2u));
        return (a ? 1u : 0u) | (b ? 2u : 0u);
    }

    __device__ __forceinline__ TileBase<I> seek(I t) {
        if (lane < h) {
            if constexpr (sizeof(I) == 4) {
                const uint32_t q1 = fast_div((uint32_t)t, mC, lC);
                x = (I)(q1 - fast_div(q1, mD, lD) * (uint32_t)d);
            } else {
                x = (t / cC) % d;
            }
        }
        I vin = x * sIn, vout = x * sOut;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            vin += __shfl_xor_sync(0xffffffffu, vin, o);
            vout += __shfl_xor_sync(0xffffffffu, vout, o);
        }
        TileBase<I> b;
        b.in = vin;
        b.out = vout;
        b.need = need();
        return b;
    }

    __device__ __forceinline__ TileBase<I> next(const TileBase<I>& cur) {
        const uint32_t wraps = __ballot_sync(0xffffffffu, lane < h && x == d - 1);
        const int f = __ffs(~wraps) - 1;  // first digit that does not wrap (< h inside the grid)
        TileBase<I> b;
        b.in = cur.in + __shfl_sync(0xffffffffu, cIn, f);
        b.out = cur.out + __shfl_sync(0xffffffffu, cOut, f);
        if (lane < f) x = 0;
        else if (lane == f) x += 1;
        b.need = need();
        return b;
    }
};

// Tile-base entry of one tile (Algorithm 1 over the grid dims, P:L84-103,
// computed by one lane with multiply-shift division): x = input offset, y =
// output offset, z = ragged state (2 bits) | interior << 2 (vector-gather
// plans: the tile's 16-byte chunks stay >= 32 bytes inside the input).
// Kernels with an interleaved tile schedule (tile t0 + it*G) keep these in a
// shared ring filled 32 tiles at a time by one warp, so a tile costs every
// warp one 16-byte shared load instead of a warp-wide Algorithm-1 decode.
__device__ __forceinline__ uint4 tile_entry(const TileParams& p, uint32_t t) {
    uint32_t vin = 0, vout = 0, need = 0;
    for (int g = 0; g < p.h; ++g) {
        const uint32_t q1 = fast_div(t, p.gMC[g], p.gLC[g]);
        const uint32_t x = q1 - fast_div(q1, p.gMD[g], p.gLD[g]) * (uint32_t)p.gD[g];
        vin += x * (uint32_t)p.gSin[g];
        vout += x * (uint32_t)p.gSout[g];
        if (x == (uint32_t)p.gD[g] - 1) {
            if (p.nSplit > 0 && g == p.splitLane[0] && p.splitTail[0] != p.splitChunk[0]) need |= 1u;
            if (p.nSplit > 1 && g == p.splitLane[1] && p.splitTail[1] != p.splitChunk[1]) need |= 2u;
        }
    }
    uint32_t interior = 0;
    if (p.vgE > 0) {
        const int64_t lo = (int64_t)vin * p.vgE;
        const int64_t hi = ((int64_t)vin + p.vgSpanIn) * p.vgE;
        interior = (lo >= 32 && hi + 32 <= p.vgInBytes) ? 4u : 0u;
    }
    return make_uint4(vin, vout, need | interior, 0u);
}

// Stateless Algorithm-1 decode for the 2-D kernels' interleaved tile order:
// each lane reads its grid dim's values from the parameter block per tile.
// (Keeping them in registers, as the walker does, measured 3.5 % slower on
// S1: it raises the 2-D kernels' register count and delays their loads;
// A/B in one process, tools/ab_lib.py.)
template <typename I, typename P>
__device__ __forceinline__ TileBase<I> decode_tile(const P& p, I t, int lane) {
    I vin = 0, vout = 0;
    bool ragged = false;
    if (lane < p.h) {
        I q;
        if constexpr (sizeof(I) == 4) {
            const uint32_t q1 = fast_div((uint32_t)t, p.gMC[lane], p.gLC[lane]);
            const uint32_t q2 = fast_div(q1, p.gMD[lane], p.gLD[lane]);
            q = (I)(q1 - q2 * (uint32_t)p.gD[lane]);
        } else {
            q = (t / (I)p.gC[lane]) % (I)p.gD[lane];
        }
        vin = q * (I)p.gSin[lane];
        vout = q * (I)p.gSout[lane];
        ragged = (q == (I)p.gD[lane] - 1) &&
                 ((p.nSplit > 0 && lane == p.splitLane[0] && p.splitTail[0] != p.splitChunk[0]) ||
                  (p.nSplit > 1 && lane == p.splitLane[1] && p.splitTail[1] != p.splitChunk[1]));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        vin += __shfl_xor_sync(0xffffffffu, vin, o);
        vout += __shfl_xor_sync(0xffffffffu, vout, o);
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, ragged);
    uint32_t need = 0;
    if (p.nSplit > 0) need |= (bal >> p.splitLane[0]) & 1u;
    if (p.nSplit > 1) need |= ((bal >> p.splitLane[1]) & 1u) << 1;
    TileBase<I> b;
    b.in = vin;
    b.out = vout;
    b.need = need;
    return b;
}

// Per slot r (tile element k = tid + r*NT): Eq. (4) global input offset,
// Eq. (5) global output offset, staging byte offsets of the load element and
// of the store element (Eq. (6) with padded strides), ragged-chunk flags.
// Slots past the tile volume (k >= V) are idle (nmine).
template <typename W, int NREG, typename I, typename FlagT>
__device__ __forceinline__ void build_slots(const TileParams& p, int tid, int NT, int nmine,
                                            I (&gin)[NREG], I (&gout)[NREG], uint32_t (&spk)[NREG],
                                            FlagT& flags) {
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        gin[r] = 0;
        gout[r] = 0;
        spk[r] = 0;
        if (r < nmine) {
            const int k = tid + r * NT;
            uint32_t f = 0;
            // Eq. (4): pMinorIn(k), tile-input order
            int rem = k;
            I off = 0;
            int sp = 0;
#pragma unroll 1  // setup, once per thread: keep the code small
            for (int i = 0; i < p.a; ++i) {
                const int c = rem % p.tExt[i];
                rem /= p.tExt[i];
                off += (I)c * (I)p.tSin[i];
                sp += c * p.tSm[i];
                if (p.nSplit > 0 && i == p.splitTile[0] && c < p.splitTail[0]) f |= 1u;
                if (p.nSplit > 1 && i == p.splitTile[1] && c < p.splitTail[1]) f |= 2u;
            }
            gin[r] = off;
            spk[r] = (uint32_t)sp * (uint32_t)sizeof(W);
            // Eqs. (5), (6): pMinorOut(k') and pSh(k'), tile-output order
            rem = k;
            off = 0;
            int sh = 0;
#pragma unroll 1
            for (int jj = 0; jj < p.a; ++jj) {
                const int t = p.tOutOrder[jj];
                const int c = rem % p.tExt[t];
                rem /= p.tExt[t];
                off += (I)c * (I)p.tSout[t];
                sh += c * p.tSm[t];
                if (p.nSplit > 0 && t == p.splitTile[0] && c < p.splitTail[0]) f |= 4u;
                if (p.nSplit > 1 && t == p.splitTile[1] && c < p.splitTail[1]) f |= 8u;
            }
            gout[r] = off;
            spk[r] |= ((uint32_t)sh * (uint32_t)sizeof(W)) << 16;
            flags |= (FlagT)f << (4 * r);
        }
    }

}

// Per-thread slot validity masks, one NREG-bit field per ragged state
// need = 0..3 (bit n*NREG + r: slot r is valid when the tile's `need` is n):
// the per-tile test becomes one shift and the per-slot test one bit test,
// instead of extracting and comparing 4 flag bits per slot.
template <int NREG, typename FlagT, typename MaskT>
__device__ __forceinline__ void slot_masks(FlagT flags, int nmine, MaskT& lm, MaskT& sm) {
    lm = 0;
    sm = 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        if (r >= nmine) continue;
        const uint32_t f = (uint32_t)(flags >> (4 * r)) & 15u;
#pragma unroll
        for (uint32_t n = 0; n < 4; ++n) {
            if ((f & n) == n) lm |= (MaskT)1 << (n * NREG + r);
            if (((f >> 2) & n) == n) sm |= (MaskT)1 << (n * NREG + r);
        }
    }
}

// Output store of the staged element: plain (out = v) or, for accumulate
// plans (f-3; "read input, read output, accumulate, write output"),
// out = alpha*v + beta*out in the element's float type with round-to-nearest
// multiplies and add and no FMA contraction (bit-exact against the oracle's
// separate operations); beta == 0 does not read out (BLAS convention).
template <typename W> struct FloatOf;
template <> struct FloatOf<uint32_t> {
    typedef float T;
    static __device__ __forceinline__ float from(uint32_t w) { return __uint_as_float(w); }
    static __device__ __forceinline__ uint32_t to(float f) { return __float_as_uint(f); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <> struct FloatOf<uint64_t> {
    typedef double T;
    static __device__ __forceinline__ double from(uint64_t w) { return __longlong_as_double((long long)w); }
    static __device__ __forceinline__ uint64_t to(double f) { return (uint64_t)__double_as_longlong(f); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct FloatOf<uint4> {  // never instantiated with ACC (no widening for accumulate)
    typedef float T;
    static __device__ __forceinline__ float from(uint4) { return 0.f; }
    static __device__ __forceinline__ uint4 to(float) { return make_uint4(0, 0, 0, 0); }
    static __device__ __forceinline__ float mul(float a, float) { return a; }
    static __device__ __forceinline__ float add(float a, float) { return a; }
};

template <typename W, int ACC>
__device__ __forceinline__ void put_out(W* dst, W v, W old, const TileParams& p) {
    if constexpr (ACC == 0) {
        stg_(dst, v);
    } else {
        typedef FloatOf<W> F;
        const typename F::T alpha = (typename F::T)p.alpha, beta = (typename F::T)p.beta;
        typename F::T r = F::mul(alpha, F::from(v));
        if (!p.betaZero) r = F::add(r, F::mul(beta, F::from(old)));
        stg_(dst, F::to(r));
    }
}

// ---------------------------------------------------------------------------
// generic staged tile, asynchronous-copy pipeline: the loads go straight from
// global to the staging buffer with cp.async (LDGSTS), no data registers, so
// S-1 tiles are in flight per CTA (S stages of shared memory) instead of one.
// Same slot tables, walker and staging layout as tile_kernel.
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void cp_async(uint32_t saddr, const void* g) {
    if constexpr (N == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(saddr), "l"(g), "n"(N));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// ---------------------------------------------------------------------------
// generic staged tile, slot-dim variant.  Same tiles, grid walk, staging
// layout and double-buffered register pipeline as tile_kernel, but a
// different thread -> element map per phase: in the load phase every thread
// owns R consecutive elements along one tile dim sL that lies outside the
// input run (so a warp still reads along the run), in the store phase R
// consecutive elements along a tile dim sS outside the output run.  Slot r of
// a pass sits at the pass base + r * (stride of the slot dim) on both the
// global and the staging side, so the per-slot tables of tile_kernel (three
// registers per element: Eq. (4) offset, Eq. (5) offset, Eq. (6) staging
// offsets) shrink to a few registers per pass of R elements.  The freed
// registers buy occupancy, i.e. loads in flight per SM (the MWP/MLP terms of
// P:L175-219 on B200).  Remaining dims + the chunk index of the slot dim form
// the phase's thread space, decoded once per thread (Eqs. 4-6).
// Validity (ragged split chunks, and a slot-dim extent that R does
// not divide) is always a prefix r < cnt of a pass; cnt is kept per pass for
// the four ragged states need = 0..3 (8 bits each).
// ---------------------------------------------------------------------------
template <typename W, int QM, int RM>
__device__ __forceinline__ void build_sd_phase(const TileParams& p, int ph, int tid, int NT,
                                               uint32_t (&g)[QM], uint32_t (&smp)[QM],
                                               uint32_t (&cnt)[QM]) {
    const int sl = p.sdSlot[ph];
    const int R = p.sdR[ph];
#pragma unroll
    for (int q = 0; q < QM; ++q) {
        g[q] = 0;
        cnt[q] = 0;
        const int u = tid + q * NT;
        if (q >= p.sdQ[ph] || u >= p.sdU[ph]) continue;
        int rem = u;
        uint32_t off = 0, sp = 0;
        int xs = 0;         // slot-dim coordinate of slot 0
        uint32_t bad = 0;   // ragged states (split bits) under which this pass is idle
#pragma unroll 1  // setup, once per thread: keep the code small
        for (int jj = 0; jj < p.a; ++jj) {
            const int t = ph == 0 ? jj : p.tOutOrder[jj];
            const int e = (t == sl) ? p.sdC[ph] : p.tExt[t];
            int c = rem % e;
            rem /= e;
            if (t == sl) {
                c *= R;
                xs = c;
            } else {
                if (p.nSplit > 0 && t == p.splitTile[0] && c >= p.splitTail[0]) bad |= 1u;
                if (p.nSplit > 1 && t == p.splitTile[1] && c >= p.splitTail[1]) bad |= 2u;
            }
            off += (uint32_t)c * (uint32_t)(ph == 0 ? p.tSin[t] : p.tSout[t]);
            sp += (uint32_t)c * (uint32_t)p.tSm[t];
        }
        g[q] = off;
        if (ph == 0) smp[q] = sp * (uint32_t)sizeof(W);
        else smp[q] |= (sp * (uint32_t)sizeof(W)) << 16;
        for (uint32_t n = 0; n < 4; ++n) {
            if (bad & n) continue;
            int lim = p.tExt[sl];
            if (p.nSplit > 0 && sl == p.splitTile[0] && (n & 1u)) lim = p.splitTail[0];
            if (p.nSplit > 1 && sl == p.splitTile[1] && (n & 2u)) lim = p.splitTail[1];
            const int k = min(max(lim - xs, 0), R);
            cnt[q] |= (uint32_t)k << (8 * n);
        }
    }
}

// ---------------------------------------------------------------------------
// row copy: fastest dim unchanged with long rows (TiledCopy class, P:L141:
// "no need for shared memory buffer since no transpose takes place")
// ---------------------------------------------------------------------------
template <typename I>
__device__ __forceinline__ I warp_sum(I v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
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

}  // namespace tt
