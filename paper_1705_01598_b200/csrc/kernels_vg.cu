// kernels_vg.cu -- generic staged tile, vector-gather load phase.
//
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
//
// The tile, its grid and its store phase are the generic tile's (Packed /
// PackedSplit classes; Eqs. 4-6; Algorithm 1,
// P:L84-103).  What changes is how the input reaches shared memory and how
// little work each element costs.
//
// Load phase.  Inside a tile the input is a set of contiguous RUNS: the
// tile's first vgM dims are the first input dims (M_m of P:L66), so run r --
// one coordinate of the remaining tile dims -- is vgL consecutive input
// elements.  Runs start at arbitrary element offsets, so a 4- or 8-byte
// gather classically moves one element per instruction and per in-flight
// register.  Here every run is copied as the 16-byte-aligned superset of its
// bytes: chunk c of run r is one cp.async.cg of 16 bytes (LDGSTS.128) when
// 16c < shift + run bytes, where shift = the run start's offset inside its
// 16-byte chunk.  The superset never leaves the run's 32-byte sectors, so
// DRAM traffic is unchanged.  Chunks of tiles touching the first or last 32
// bytes of the input are copied element by element (no read outside the
// tensor).  No data registers: S-1 tiles are in flight per CTA.
//
// Shift folding.  shift_r = (sh + q_r) mod 16 with sh = the tile base's
// offset inside its chunk and q_r = the run offset's (both multiples of E).
// The load places chunk 0 of run r at slot_r + 16 w_r, w_r = [sh + q_r >= 16]
// (equivalently shift_r < q_r), so element i of run r is ALWAYS at
// slot_r + q_r + i*E + sh: the store phase adds one per-tile constant.
//
// Per-element cost.  Each thread owns K fixed (run, chunk) load items and
// NREG fixed output-order store slots (tables computed once); the tile bases
// (Algorithm 1) are decoded 32 tiles at a time by one warp into a shared
// ring, so a tile costs every warp one 16-byte shared load.  A store slot is
// LDS + IMAD.WIDE + STG + one add; ragged tiles predicate the STG
// per slot instead of branching.
//
// Pipeline: S stages, S-1 tiles in flight; per stage a "full" mbarrier (the
// copies have landed: cp.async.mbarrier.arrive) and an "empty" one (every
// warp has read it), so warps wait only for data and for the slowest reader
// of the stage being refilled -- no CTA-wide barrier per tile.
//
// Shared memory: S stages of p.sbuf elements, then the tile-base ring (128 x
// uint4: input offset, output offset, ragged state | interior << 2), then
// the 2 S mbarriers.
#include "kern_common.cuh"
#include "kern_pick.h"

namespace tt {

__device__ __forceinline__ void stg_pred(uint32_t* p, uint32_t v, bool ok) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.global.b32 [%0], %1; }" ::"l"(p), "r"(v),
                 "r"((uint32_t)ok)
                 : "memory");
}
__device__ __forceinline__ void stg_pred(uint64_t* p, uint64_t v, bool ok) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.global.b64 [%0], %1; }" ::"l"(p), "l"(v),
                 "r"((uint32_t)ok)
                 : "memory");
}
// Cache flavour of the 16-byte chunk copies (p.vgPolicy): 0 = .ca (through
// L1), 1 = .cg (L2 only).  Measured (profiles/round2_vg_policy.txt): with .cg
// the L1 does not merge the 16-byte requests of one 32-byte sector, so L2
// sees ~1.5x the sector requests and DRAM re-reads the sectors shared by
// neighbouring runs (+24 % read traffic on 5^12 fp32); .ca is the default.
template <int POL>
__device__ __forceinline__ void cp_async16_pred(uint32_t saddr, const void* g, bool ok) {
    if constexpr (POL == 0)
        asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.ca.shared.global [%0], [%1], 16; }" ::"r"(saddr),
                     "l"(g), "r"((uint32_t)ok));
    else
        asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(saddr),
                     "l"(g), "r"((uint32_t)ok));
}

// mbarrier pipeline (per stage: "full" = the stage's copies have landed,
// count NT, one asynchronous arrive per thread after its copies; "empty" =
// every warp has read the stage, count = warps)
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(a) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t a) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

// Launch bound: up to 512 threads with 16 store slots; with fewer slots a
// "wide" instantiation for up to 1024 threads (64 registers) and a narrow
// one for up to 768 (85 registers: room to keep the per-tile pipeline
// addresses instead of recomputing them), picked by the plan's thread count.
template <typename W, int NREG, int K, int S, bool WIDE>
__global__ void __launch_bounds__(NREG >= 16 ? 512 : (WIDE ? 1024 : 768), 1)
tile_vg_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    constexpr uint32_t E = sizeof(W);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * E;
    uint4* const ring = reinterpret_cast<uint4*>(smem_raw + p.vgTab);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int M = p.vgM;
    const uint32_t nch = (uint32_t)p.vgNch;

    // --- load items: item k = (run r, chunk c), u = tid + k*NT -----------------
    // roff = (run offset in bytes from the tile base, Eq. 4 over the non-run
    // dims, rounded down to 16) + 16c, with q_r = that offset mod 16 in its
    // low 4 bits; pk = slot byte offset + 16c (bits 0-17) | validity in the
    // four ragged states (18-21) | c (24-31).  Per tile, with sh = the tile
    // base's offset inside its 16-byte chunk: t = sh + q_r, the chunk's source
    // is the tile base rounded down to 16 + (roff - q_r) + (t & 16), its
    // staging slot + (t & 16), its run's shift t & 15.
    uint32_t roff[K], pk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        roff[k] = 0;
        pk[k] = 0;
        const uint32_t u = (uint32_t)tid + (uint32_t)k * (uint32_t)NT;
        if (u < (uint32_t)p.vgNR * nch) {
            const uint32_t r = u / nch, c = u - r * nch;
            uint32_t rem = r, off = 0, smb = 0, bad = 0;
#pragma unroll 1  // setup, once per thread: keep the code small
            for (int t = M; t < p.a; ++t) {
                const uint32_t x = rem % (uint32_t)p.tExt[t];
                rem /= (uint32_t)p.tExt[t];
                off += x * (uint32_t)p.tSin[t];
                smb += x * (uint32_t)p.tSm[t];
                if (p.nSplit > 0 && t == p.splitTile[0] && x >= (uint32_t)p.splitTail[0]) bad |= 1u;
                if (p.nSplit > 1 && t == p.splitTile[1] && x >= (uint32_t)p.splitTail[1]) bad |= 2u;
            }
            uint32_t valid = 0;
            for (uint32_t n = 0; n < 4; ++n)
                if ((bad & n) == 0) valid |= 1u << n;
            roff[k] = (off * E & ~15u) + 16u * c + ((off * E) & 15u);
            pk[k] = (smb * E + 16u * c) | (valid << 18) | (c << 24);
        }
    }

    // --- store slots: element k' = tid + r*NT in tile-output order ---------------
    // gout = Eq. (5) offset; spk = slot_r + q_r + in-run index * E (Eq. 6 with
    // the run layout and the folded shift); m<n> = slots valid in state n
    uint32_t gout[NREG], spk[NREG];
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        gout[r] = 0;
        spk[r] = 0;
        const int kk = tid + r * NT;
        if (kk < p.V) {
            int rem = kk;
            uint32_t go = 0, inrun = 0, smb = 0, ro = 0, f = 0;
#pragma unroll 1  // setup, once per thread: keep the code small
            for (int jj = 0; jj < p.a; ++jj) {
                const int t = p.tOutOrder[jj];
                const uint32_t x = (uint32_t)(rem % p.tExt[t]);
                rem /= p.tExt[t];
                go += x * (uint32_t)p.tSout[t];
                if (t < M) {
                    inrun += x * (uint32_t)p.tCin[t];
                } else {
                    smb += x * (uint32_t)p.tSm[t];
                    ro += x * (uint32_t)p.tSin[t];
                }
                if (p.nSplit > 0 && t == p.splitTile[0] && x < (uint32_t)p.splitTail[0]) f |= 1u;
                if (p.nSplit > 1 && t == p.splitTile[1] && x < (uint32_t)p.splitTail[1]) f |= 2u;
            }
            gout[r] = go;
            spk[r] = (smb + inrun) * E + ((ro * E) & 15u);
            m0 |= 1u << r;
            if (f & 1u) m1 |= 1u << r;
            if (f & 2u) m2 |= 1u << r;
            if ((f & 3u) == 3u) m3 |= 1u << r;
        }
    }
    const uint32_t full = (1u << NREG) - 1u;

    const uint32_t nTiles = (uint32_t)p.nTiles;
    const uint32_t G = (uint32_t)gridDim.x;
    const uint32_t t0 = (uint32_t)blockIdx.x;
    if (t0 >= nTiles) return;
    const uint32_t nIt = (nTiles - t0 + G - 1) / G;  // tiles of this CTA: t0 + it*G
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t fullB = sm0 + (uint32_t)p.vgTab + 128u * 16u;  // full[s] at fullB + 8 s
    const uint32_t emptyB = fullB + 8u * S;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(fullB + 8u * s, (uint32_t)NT);
            mbar_init(emptyB + 8u * s, (uint32_t)(NT >> 5));
        }
    }
    if (warp == 0) {  // tile bases of iterations 0..63
        for (uint32_t it = (uint32_t)lane; it < 64u && it < nIt; it += 32)
            ring[it] = tile_entry(p, t0 + it * G);
    }
    __syncthreads();

    const char* const inB = reinterpret_cast<const char*>(in);
    const uint32_t LB = (uint32_t)p.vgL * E, LtB = (uint32_t)p.vgLtail * E;
    const uint32_t runBit = (uint32_t)p.vgRunBit;
    const int pol = p.vgPolicy;

    auto issue = [&](uint32_t it, uint32_t sb) {
        const uint4 e = ring[it & 127u];
        const uint32_t nd = e.z & 3u;
        const uint32_t Lb = (runBit & nd) ? LtB : LB;
        const char* const tb = inB + (size_t)e.x * E;
        const uint32_t vs = 18u + nd;
        if (e.z & 4u) {
            const uint32_t sh = (uint32_t)reinterpret_cast<uintptr_t>(tb) & 15u;
            const char* const tbA = tb - sh;
            const uint32_t vmask = 1u << vs;
            auto items = [&](auto polc) {
                constexpr int POL = decltype(polc)::value;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const uint32_t q = roff[k] & 15u;
                    const uint32_t t = sh + q;
                    const uint32_t cy = t & 16u;       // the run's first byte is in the next chunk
                    const uint32_t c16 = (pk[k] >> 20) & 0xff0u;
                    const bool ok = (pk[k] & vmask) && c16 < (t & 15u) + Lb;
                    const uint32_t dst = sb + (pk[k] & 0x3ffffu) + cy;
                    cp_async16_pred<POL>(dst, tbA + (roff[k] - q + cy), ok);
                }
            };
            if (pol == 1) items(std::integral_constant<int, 1>());
            else items(std::integral_constant<int, 0>());
        } else {  // near an end of the input: element-wise inside the tensor
            const char* const lo = inB;
            const char* const hi = inB + p.vgInBytes;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t q = roff[k] & 15u;
                const uint32_t c16 = (pk[k] >> 20) & 0xff0u;
                const char* a = tb + (roff[k] - q - c16) + q;   // the run's first byte
                const uint32_t s = (uint32_t)reinterpret_cast<uintptr_t>(a) & 15u;
                if (!(((pk[k] >> vs) & 1u) && c16 < s + Lb)) continue;
                const uint32_t dst = sb + (pk[k] & 0x3ffffu) + (s < q ? 16u : 0u);
                const char* src = a - s + c16;
                if (src >= lo && src + 16 <= hi) {
                    cp_async<16>(dst, src);
                } else {
#pragma unroll
                    for (uint32_t j = 0; j < 16u / E; ++j)
                        if (src + j * E >= lo && src + j * E < hi) cp_async<E>(dst + j * E, src + j * E);
                }
            }
        }
    };

#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        if ((uint32_t)s < nIt) {
            issue((uint32_t)s, sm0 + (uint32_t)s * sbytes);
            cp_async_mbar_arrive(fullB + 8u * s);
        }
    }
    uint32_t stage = 0;
    for (uint32_t it = 0; it < nIt; ++it) {
        mbar_wait(fullB + 8u * stage, (it / S) & 1u);   // tile it has landed in its stage
        if ((it & 31u) == 0 && it >= 32u && warp == 0) {  // tile bases of iterations it+32 .. it+63
            const uint32_t j = it + 32u + (uint32_t)lane;
            if (j < nIt) ring[j & 127u] = tile_entry(p, t0 + j * G);
        }
        // transposed read of the staged tile (Eq. 6), coalesced writes (Eq. 5)
        {
            const uint4 e = ring[it & 127u];
            const uint32_t nd = e.z & 3u;
            const uint32_t sbsh = sm0 + stage * sbytes +
                                  ((uint32_t)reinterpret_cast<uintptr_t>(inB + (size_t)e.x * E) & 15u);
            W* const dst = out + e.y;
            const uint32_t m = nd == 0 ? m0 : nd == 1 ? m1 : nd == 2 ? m2 : m3;
            if (m == full) {
#pragma unroll
                for (int r = 0; r < NREG; ++r) stg_(elem_addr(dst, gout[r]), lds<W>(sbsh + spk[r]));
            } else {
#pragma unroll
                for (int r = 0; r < NREG; ++r)
                    stg_pred(elem_addr(dst, gout[r]), lds<W>(sbsh + spk[r]), (m & (1u << r)) != 0u);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(emptyB + 8u * stage);
        // refill the stage read in the previous iteration with tile it+S-1,
        // once every warp has read it
        const uint32_t itn = it + (uint32_t)(S - 1);
        if (itn < nIt) {
            const uint32_t sn = (stage == 0) ? (uint32_t)(S - 1) : stage - 1;
            if (itn >= (uint32_t)S) mbar_wait(emptyB + 8u * sn, ((itn - S) / S) & 1u);
            issue(itn, sm0 + sn * sbytes);
            cp_async_mbar_arrive(fullB + 8u * sn);
        }
        stage = (stage + 1 == (uint32_t)S) ? 0u : stage + 1;
    }
}

// vector-gather tile: 4/8-byte words, NREG store slots in {4, 8, 16}, K load
// items in {2, 3, 4}, 3 or 4 stages, 32-bit indices; threads picks the launch
// bound (above; 16-slot plans have one)
template <typename W, int R, int S, bool WD>
static const void* pick_vg_k(int items) {
    if (items <= 2) return (const void*)&tile_vg_kernel<W, R, 2, S, WD>;
    if (items <= 3) return (const void*)&tile_vg_kernel<W, R, 3, S, WD>;
    if (items <= 4) return (const void*)&tile_vg_kernel<W, R, 4, S, WD>;
    return nullptr;
}
template <typename W, int S>
static const void* pick_vg_r(int nreg, int items, int threads) {
    const bool wide = threads > 768;
    switch (nreg) {
        case 4: return wide ? pick_vg_k<W, 4, S, true>(items) : pick_vg_k<W, 4, S, false>(items);
        case 8: return wide ? pick_vg_k<W, 8, S, true>(items) : pick_vg_k<W, 8, S, false>(items);
        case 16: return pick_vg_k<W, 16, S, false>(items);
        default: return nullptr;
    }
}
const void* pick_tile_vg(int esize, int nreg, int items, int stages, int threads) {
    if (esize == 4) {
        if (stages == 3) return pick_vg_r<uint32_t, 3>(nreg, items, threads);
        if (stages == 4) return pick_vg_r<uint32_t, 4>(nreg, items, threads);
    } else if (esize == 8) {
        if (stages == 3) return pick_vg_r<uint64_t, 3>(nreg, items, threads);
        if (stages == 4) return pick_vg_r<uint64_t, 4>(nreg, items, threads);
    }
    return nullptr;
}

}  // namespace tt
