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
#include <mutex>
#include <type_traits>
#include <unordered_set>

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
    __device__ __forceinline__ GridWalker(const P& p, int lane_) : lane(lane_) {
        h = p.h;
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

// Per slot r (tile element k = tid + r*NT): gin/gout = global minor offsets
// (Eqs. 4, 5), sin/sout = staging byte offsets of the load element and of the
// store element (Eq. 6 through the padded layout).  `flags` holds 4 bits per
// slot: (load elem inside ragged A-chunk, ... B-chunk, store elem inside
// ragged A-chunk, ... B-chunk); a slot is valid in a ragged tile iff its bits
// cover the tile's `need`.
template <typename W, int NREG, typename I, int ACC = 0>
__global__ void __launch_bounds__(NREG >= 16 ? 256 : 512, (NREG >= 16 ? 2 : (sizeof(I) == 8 || (NREG >= 8 && sizeof(W) >= 8) ? 1 : 2)))
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
    GridWalker<I> walk(p, lane);

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
    TileBase<I> cur = walk.seek(t0);
    load(cur);
    load_out(cur);

    uint32_t sb = sm0;
    for (I t = t0; t < t1; t += step) {
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
        // issue the next tile's global loads before writing this one
        const TileBase<I> now = cur;
        if (t + step < t1) {
            cur = il ? walk.seek(t + step) : walk.next(cur);
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
    GridWalker<uint32_t> walk(p, lane);

    W v[QM][RM];
    auto load = [&](const TileBase<uint32_t>& tb) {
        const uint32_t sh = 8u * tb.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QL) break;
            const uint32_t c = (cntL[q] >> sh) & 0xffu;
            const W* __restrict__ src = opaque(in + tb.in + gin[q]);
            if (c == (uint32_t)RM) {
#pragma unroll
                for (int r = 0; r < RM; ++r) v[q][r] = ldg_(elem_addr(src, (uint32_t)r * sIn));
            } else {
#pragma unroll
                for (int r = 0; r < RM; ++r)
                    if ((uint32_t)r < c) v[q][r] = ldg_(elem_addr(src, (uint32_t)r * sIn));
            }
        }
    };
    TileBase<uint32_t> cur = walk.seek(t0);
    load(cur);

    uint32_t sb = sm0;
    for (uint32_t t = t0; t < nTiles; t += G) {
        // stage the tile (input-side map)
        {
            const uint32_t sh = 8u * cur.need;
#pragma unroll
            for (int q = 0; q < QM; ++q) {
                if (q >= QL) break;
                const uint32_t c = (cntL[q] >> sh) & 0xffu;
                const uint32_t a0 = sb + (smp[q] & 0xffffu);
#pragma unroll
                for (int r = 0; r < RM; ++r)
                    if ((uint32_t)r < c) sts(a0 + (uint32_t)r * mIn, v[q][r]);
            }
        }
        __syncthreads();
        const TileBase<uint32_t> now = cur;
        if (t + G < nTiles) {
            cur = walk.seek(t + G);
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
                const uint32_t a0 = sb + (smp[q] >> 16);
                if (c == (uint32_t)RM) {
#pragma unroll
                    for (int r = 0; r < RM; ++r)
                        stg_(elem_addr(dst, (uint32_t)r * sOut), lds<W>(a0 + (uint32_t)r * mOut));
                } else {
#pragma unroll
                    for (int r = 0; r < RM; ++r)
                        if ((uint32_t)r < c)
                            stg_(elem_addr(dst, (uint32_t)r * sOut), lds<W>(a0 + (uint32_t)r * mOut));
                }
            }
        }
        sb = (sb == sm0) ? sm0 + sbytes : sm0;
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
    GridWalker<uint32_t> walk(p, lane);

    // load phase of tile t into the staging buffer at byte address sb
    auto issue = [&](uint32_t t, uint32_t sb) {
        const TileBase<uint32_t> tb = walk.seek(t);
        const uint32_t sh = 8u * tb.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QL) break;
            const uint32_t c = (cntL[q] >> sh) & 0xffu;
            const W* src = in + tb.in + gin[q];
            const uint32_t a0 = sb + (smp[q] & 0xffffu);
#pragma unroll
            for (int r = 0; r < RM; ++r)
                if ((uint32_t)r < c) cp_async<sizeof(W)>(a0 + (uint32_t)r * mIn, elem_addr(src, (uint32_t)r * sIn));
        }
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        const uint32_t t = t0 + (uint32_t)s * G;
        if (t < nTiles) issue(t, sm0 + (uint32_t)s * sbytes);
        cp_async_commit();
    }
    uint32_t k = 0;
    for (uint32_t t = t0; t < nTiles; t += G) {
        cp_async_wait<S - 2>();
        __syncthreads();
        // refill the stage read in the previous iteration (all threads are
        // past its reads: they passed this iteration's barrier)
        {
            const uint32_t tn = t + (uint32_t)(S - 1) * G;
            const uint32_t kn = (k + S - 1) % S;
            if (tn < nTiles) issue(tn, sm0 + kn * sbytes);
            cp_async_commit();
        }
        const TileBase<uint32_t> now = walk.seek(t);
        const uint32_t sb = sm0 + k * sbytes;
        const uint32_t sh = 8u * now.need;
#pragma unroll
        for (int q = 0; q < QM; ++q) {
            if (q >= QS) break;
            const uint32_t c = (cntS[q] >> sh) & 0xffu;
            W* __restrict__ dst = opaque(out + now.out + gout[q]);
            const uint32_t a0 = sb + (smp[q] >> 16);
            if (c == (uint32_t)RM) {
#pragma unroll
                for (int r = 0; r < RM; ++r)
                    stg_(elem_addr(dst, (uint32_t)r * sOut), lds<W>(a0 + (uint32_t)r * mOut));
            } else {
#pragma unroll
                for (int r = 0; r < RM; ++r)
                    if ((uint32_t)r < c)
                        stg_(elem_addr(dst, (uint32_t)r * sOut), lds<W>(a0 + (uint32_t)r * mOut));
            }
        }
        k = (k + 1 == (uint32_t)S) ? 0u : k + 1;
    }
    cp_async_wait<0>();
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
    const I L = (I)p.row;

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
    for (I r = r0; r < r1; ++r) {
        const W* __restrict__ src = opaque(in + base);
        W* __restrict__ dst = opaque(out + r * L);
        for (I c = lane; c < L; c += 32 * U) {
            W t[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c + 32 * u < L) t[u] = ldg_(src + c + 32 * u);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c + 32 * u < L) stg_(dst + c + 32 * u, t[u]);
        }
        // odometer step to row r+1
        const uint32_t wraps = __ballot_sync(0xffffffffu, lane < p.h && x == d - 1);
        const int f = __ffs(~wraps) - 1;
        I delta = 0;
        if (lane < f) { delta = (I)0 - (d - 1) * s; x = 0; }
        else if (lane == f) { delta = s; x += 1; }
        base += warp_sum<I>(delta);
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

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
// slot-dim variant: (passes, slots) in {(1,16), (2,8), (4,4)}, 4/8-byte words,
// 32-bit indices
static const void* pick_tile_sd(int esize, int q, int r, int stages = 0) {
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

template <typename W, int NREG, typename I>
static const void* tile_fn() {
    return reinterpret_cast<const void*>(&tile_kernel<W, NREG, I>);
}

// accumulate variant (f-3): 4/8-byte words, 32-bit indices
static const void* pick_tile_acc(int esize, int nreg) {
#define TT_PICKACC(W)                                                               \
    switch (nreg) {                                                                 \
        case 1: return (const void*)&tile_kernel<W, 1, uint32_t, 1>;               \
        case 2: return (const void*)&tile_kernel<W, 2, uint32_t, 1>;               \
        case 4: return (const void*)&tile_kernel<W, 4, uint32_t, 1>;               \
        case 8: return (const void*)&tile_kernel<W, 8, uint32_t, 1>;               \
        case 16: return (const void*)&tile_kernel<W, 16, uint32_t, 1>;             \
        default: return nullptr;                                                    \
    }
    if (esize == 4) { TT_PICKACC(uint32_t) }
    if (esize == 8) { TT_PICKACC(uint64_t) }
    return nullptr;
#undef TT_PICKACC
}

static const void* pick_tile(int esize, int nreg, bool idx64) {
#define TT_PICK(W, I)                               \
    switch (nreg) {                                 \
        case 1: return tile_fn<W, 1, I>();          \
        case 2: return tile_fn<W, 2, I>();          \
        case 4: return tile_fn<W, 4, I>();          \
        case 8: return tile_fn<W, 8, I>();          \
        case 16: return tile_fn<W, 16, I>();        \
        default: return nullptr;                    \
    }
    if (esize == 4) {
        if (idx64) { TT_PICK(uint32_t, int64_t) } else { TT_PICK(uint32_t, uint32_t) }
    } else if (esize == 8) {
        if (idx64) { TT_PICK(uint64_t, int64_t) } else { TT_PICK(uint64_t, uint32_t) }
    } else if (esize == 16) {  // widened words: at most 4 slots (register budget)
        switch (nreg) {
            case 1: return idx64 ? tile_fn<uint4, 1, int64_t>() : tile_fn<uint4, 1, uint32_t>();
            case 2: return idx64 ? tile_fn<uint4, 2, int64_t>() : tile_fn<uint4, 2, uint32_t>();
            case 4: return idx64 ? tile_fn<uint4, 4, int64_t>() : tile_fn<uint4, 4, uint32_t>();
            default: return nullptr;
        }
    }
    return nullptr;
#undef TT_PICK
}

// asynchronous-copy tile: 3 stages, 32-bit indices, 4/8/16-byte words
static const void* pick_tile_async(int esize, int nreg, bool idx64) {
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

static const void* pick_rowcopy(int esize, bool idx64) {
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
static const void* pick_tiled2d_async(int esize, int ta, int tb, int stages) {
    if (esize == 4 && ta == 64 && tb == 64) return t2dsa_fn<uint32_t, 2, 8>(stages);
    if (esize == 4 && ta == 128 && tb == 64) return t2dsa_fn<uint32_t, 4, 8>(stages);
    if (esize == 4 && ta == 64 && tb == 128) return t2dsa_fn<uint32_t, 2, 16>(stages);
    if (esize == 8 && ta == 64 && tb == 64) return t2dsa_fn<uint64_t, 2, 8>(stages);
    if (esize == 8 && ta == 32 && tb == 64) return t2dsa_fn<uint64_t, 1, 8>(stages);
    if (esize == 8 && ta == 64 && tb == 32) return t2dsa_fn<uint64_t, 2, 4>(stages);
    return nullptr;
}

static const void* pick_tiled2d(int esize, int vec, int ta, int tb, bool idx64) {
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

// Raise a kernel's dynamic shared-memory limit to the device maximum ONCE
// per function (and device).  Setting the attribute on every launch costs a
// driver call per launch and measured 4 % of S1 throughput on a non-default
// stream (back-to-back launches).
static std::mutex g_smem_mu;
static std::unordered_set<uint64_t> g_smem_done;

static cudaError_t ensure_max_smem(const void* fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t key = reinterpret_cast<uint64_t>(fn) ^ ((uint64_t)dev << 56);
    std::lock_guard<std::mutex> g(g_smem_mu);
    if (g_smem_done.count(key)) return cudaSuccess;
    int maxOptin = 0;
    e = cudaDeviceGetAttribute(&maxOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxOptin);
    if (e == cudaSuccess) g_smem_done.insert(key);
    return e;
}

int cuda_occupancy(const OccQuery& q, const DeviceInfo& dev) {
    (void)dev;
    const void* fn = q.kernel == TT_KERNEL_TILE
                         ? (q.sdq ? pick_tile_sd(q.esize, q.sdq, q.sdr, q.vec >= 3 ? q.vec : 0)
                            : q.acc ? pick_tile_acc(q.esize, q.nreg)
                                      : (q.vec >= 3 ? pick_tile_async(q.esize, q.nreg, q.idx64)
                                                    : pick_tile(q.esize, q.nreg, q.idx64)))
                     : q.kernel == TT_KERNEL_TILED2D
                         ? (q.vec == 1 && q.sdq >= 3 && !q.idx64  // sdq = stages for the 2-D ring
                                ? pick_tiled2d_async(q.esize, q.ta, q.tb, q.sdq)
                                : pick_tiled2d(q.esize, q.vec, q.ta, q.tb, q.idx64))
                     : q.kernel == TT_KERNEL_ROWCOPY ? pick_rowcopy(q.esize, q.idx64)
                                                     : nullptr;
    if (!fn) return 0;
    if (ensure_max_smem(fn) != cudaSuccess) {
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

int launch_plan(const Plan& plan0, const void* in, void* out, void* stream_) {
    return launch_plan_scaled(plan0, in, out, stream_, 1.0, 0.0);
}

int launch_plan_scaled(const Plan& plan0, const void* in, void* out, void* stream_, double alpha,
                       double beta) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    // widened words need E*widen-aligned pointers; otherwise run the narrow plan
    const Plan& plan = (plan0.widen > 1 && plan0.narrow &&
                        ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) &
                         (uintptr_t)(plan0.prob.esize - 1)) != 0)
                           ? *plan0.narrow
                           : plan0;
    const KernelChoice& kc = plan.kc;
    const int E = plan.prob.esize;
    if (kc.kernel == TT_KERNEL_COPY) {
        const int vec16 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
        const int64_t n = plan.prob.vol * (E / 4);  // copy in 4-byte words
        copy_kernel<uint32_t><<<kc.grid, kc.threads, 0, stream>>>(
            static_cast<const uint32_t*>(in), static_cast<uint32_t*>(out), n, vec16);
        return (int)cudaGetLastError();
    }
    if (kc.kernel == TT_KERNEL_ROWCOPY) {
        const void* fn = pick_rowcopy(E, kc.idx64);
        if (!fn) return (int)cudaErrorInvalidConfiguration;
        void* args[] = {(void*)&plan.row, (void*)&in, (void*)&out};
        return (int)cudaLaunchKernel(fn, dim3(kc.grid), dim3(kc.threads), args, 0, stream);
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
        const void* fn = t2 ? (kc.vec == 1 && kc.stages >= 3 && !kc.idx64
                                   ? pick_tiled2d_async(E, kc.tile0, kc.tile1, kc.stages)
                                   : pick_tiled2d(E, kc.vec, kc.tile0, kc.tile1, kc.idx64))
                            : kc.sdq ? pick_tile_sd(E, kc.sdq, kc.sdr, kc.stages)
                            : kc.acc ? pick_tile_acc(E, kc.nreg)
                                     : (kc.stages >= 3 ? pick_tile_async(E, kc.nreg, kc.idx64)
                                                       : pick_tile(E, kc.nreg, kc.idx64));
        if (!fn) return (int)cudaErrorInvalidConfiguration;
        if (smem > 48 * 1024) {
            cudaError_t e = ensure_max_smem(fn);
            if (e != cudaSuccess) return (int)e;
        }
        TileParams scaled;
        const void* pp = t2 ? (const void*)&plan.t2d : (const void*)&plan.tile;
        if (kc.acc) {
            scaled = plan.tile;
            scaled.alpha = alpha;
            scaled.beta = beta;
            scaled.betaZero = beta == 0.0;
            pp = &scaled;
        }
        void* args[] = {const_cast<void*>(pp), (void*)&in, (void*)&out};
        return (int)cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, stream);
    }
    return (int)cudaErrorInvalidConfiguration;
}

}  // namespace tt
