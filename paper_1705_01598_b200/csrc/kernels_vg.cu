// kernels_vg.cu -- generic staged tile, vector-gather load phase.
//
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
//
// The tile, grid walk and store phase are the generic tile's (Packed /
// PackedSplit classes; Eqs. 4-6; Algorithm 1,
// P:L84-103).  What changes is how the input side reaches shared memory.
// Inside a tile the input is a set of contiguous RUNS: the tile's first vgM
// dims are the first input dims (M_m of P:L66), so run r -- one coordinate of
// the remaining tile dims -- is vgL consecutive input elements.  Runs start at
// arbitrary element offsets, so 4- and 8-byte gathers classically move one
// element per instruction and per in-flight register (the loads-in-flight
// limit of section 11 in DESIGN.md).  Here every run is copied as the
// 16-byte-aligned superset of its bytes: ceil((shift + vgL*E) / 16) chunks
// of 16 bytes, each one cp.async.cg (LDGSTS.128) into the run's 16-byte-
// aligned shared-memory slot.  The run's elements then sit `shift` bytes into
// the slot (shift = the run start's offset inside its 16-byte chunk, which
// depends on the tile base and the run's offset); the store phase adds it
// back when it reads the staged tile in output order (Eq. 6) and writes
// coalesced runs (Eq. 5).  The superset never leaves the run's 32-byte
// sectors, so DRAM traffic is unchanged; chunks that would cross the ends of
// the input tensor are copied element by element.  No data registers: S-1
// tiles are in flight per CTA (an S-stage ring).
//
// Shared memory: S stages of p.sbuf elements, then the run table (uint2 per
// run: {run offset in elements from the tile base, staging byte offset |
// validity bits << 24}), built once per CTA.
#include "kern_common.cuh"
#include "kern_pick.h"

namespace tt {

template <typename W, int NREG, int S>
__global__ void __launch_bounds__(NREG >= 16 ? 256 : 1024, NREG >= 16 ? 2 : 1)
tile_vg_kernel(const __grid_constant__ TileParams p, const W* __restrict__ in, W* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t sm0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t sbytes = (uint32_t)p.sbuf * (uint32_t)sizeof(W);
    const int tid = threadIdx.x;
    const int NT = blockDim.x;
    const int lane = tid & 31;
    const int M = p.vgM;
    const int NR = p.vgNR;
    uint2* const tab = reinterpret_cast<uint2*>(smem_raw + p.vgTab);

    // run table: offset (Eq. 4 over the non-run tile dims) and staging slot
    // (Eq. 6 with the padded strides) of every run; validity per ragged state
    for (int r = tid; r < NR; r += NT) {
        int rem = r;
        uint32_t off = 0, smb = 0, bad = 0;
        for (int t = M; t < p.a; ++t) {
            const int c = rem % p.tExt[t];
            rem /= p.tExt[t];
            off += (uint32_t)c * (uint32_t)p.tSin[t];
            smb += (uint32_t)c * (uint32_t)p.tSm[t];
            if (p.nSplit > 0 && t == p.splitTile[0] && c >= p.splitTail[0]) bad |= 1u;
            if (p.nSplit > 1 && t == p.splitTile[1] && c >= p.splitTail[1]) bad |= 2u;
        }
        uint32_t valid = 0;
        for (uint32_t n = 0; n < 4; ++n)
            if ((bad & n) == 0) valid |= 1u << n;
        tab[r] = make_uint2(off, smb * (uint32_t)sizeof(W) | (valid << 24));
    }

    // store-phase slot tables: element k' = tid + r*NT in tile-output order;
    // gout = Eq. (5) offset, spk = staging byte offset (run slot + in-run
    // index) | run offset mod 16 bytes << 24, validity bits as build_slots
    uint32_t gout[NREG], spk[NREG];
    uint32_t fl = 0;  // 2 bits per slot: element inside the ragged chunk of split 0 / 1
    const int nmine = (p.V > tid) ? min(NREG, (p.V - tid + NT - 1) / NT) : 0;
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        gout[r] = 0;
        spk[r] = 0;
        if (r < nmine) {
            int rem = tid + r * NT;
            uint32_t go = 0, inrun = 0, smb = 0, roff = 0, f = 0;
            for (int jj = 0; jj < p.a; ++jj) {
                const int t = p.tOutOrder[jj];
                const int c = rem % p.tExt[t];
                rem /= p.tExt[t];
                go += (uint32_t)c * (uint32_t)p.tSout[t];
                if (t < M) {
                    inrun += (uint32_t)c * (uint32_t)p.tCin[t];
                } else {
                    smb += (uint32_t)c * (uint32_t)p.tSm[t];
                    roff += (uint32_t)c * (uint32_t)p.tSin[t];
                }
                if (p.nSplit > 0 && t == p.splitTile[0] && c < p.splitTail[0]) f |= 1u;
                if (p.nSplit > 1 && t == p.splitTile[1] && c < p.splitTail[1]) f |= 2u;
            }
            gout[r] = go;
            spk[r] = (smb + inrun) * (uint32_t)sizeof(W) | (((roff * (uint32_t)sizeof(W)) & 15u) << 24);
            fl |= f << (2 * r);
        }
    }
    uint32_t smask = 0;  // bit n*NREG + r: slot r valid when the tile's need is n
#pragma unroll
    for (int r = 0; r < NREG; ++r) {
        if (r >= nmine) continue;
        const uint32_t f = (fl >> (2 * r)) & 3u;
#pragma unroll
        for (uint32_t n = 0; n < 4; ++n)
            if ((f & n) == n && n * NREG + r < 32) smask |= 1u << (n * NREG + r);
    }
    // NREG == 16: states 2 and 3 do not fit the 32-bit mask; keep them apart
    uint32_t smaskHi = 0;
    if constexpr (NREG == 16) {
#pragma unroll
        for (int r = 0; r < NREG; ++r) {
            if (r >= nmine) continue;
            const uint32_t f = (fl >> (2 * r)) & 3u;
            if ((f & 2u) == 2u) smaskHi |= 1u << r;
            if ((f & 3u) == 3u) smaskHi |= 1u << (16 + r);
        }
    }
    __syncthreads();  // run table visible

    const uint32_t nTiles = (uint32_t)p.nTiles;
    const uint32_t G = (uint32_t)gridDim.x;
    const uint32_t t0 = (uint32_t)blockIdx.x;
    if (t0 >= nTiles) return;
    GridWalker<uint32_t> walk(p, lane);

    const int Gl = p.vgG;                 // lanes per run group
    const int grp = tid / Gl, lg = tid % Gl, nGrp = NT / Gl;
    const char* const inLo = reinterpret_cast<const char*>(in);
    const char* const inHi = inLo + p.vgInBytes;

    // load phase of tile t into the stage at byte address sb
    auto issue = [&](uint32_t t, uint32_t sb) {
        const TileBase<uint32_t> tb = walk.seek(t);
        const uint32_t nd = tb.need;
        const uint32_t Lb = ((p.vgRunBit & nd) ? (uint32_t)p.vgLtail : (uint32_t)p.vgL) * (uint32_t)sizeof(W);
        const W* const base = in + tb.in;
        for (int r = grp; r < NR; r += nGrp) {
            const uint2 e = tab[r];
            if (!((e.y >> (24 + nd)) & 1u)) continue;
            const uintptr_t ga = reinterpret_cast<uintptr_t>(base + e.x);
            const char* const g0 = reinterpret_cast<const char*>(ga & ~(uintptr_t)15);
            const uint32_t nch = ((uint32_t)(ga & 15u) + Lb + 15u) >> 4;
            const uint32_t dst = sb + (e.y & 0xffffffu);
            for (uint32_t c = (uint32_t)lg; c < nch; c += (uint32_t)Gl) {
                const char* const src = g0 + 16u * c;
                if (src >= inLo && src + 16 <= inHi) {
                    cp_async<16>(dst + 16u * c, src);
                } else {  // a chunk crossing an end of the input tensor
#pragma unroll
                    for (uint32_t k = 0; k < 16u / sizeof(W); ++k) {
                        const char* const s1 = src + k * sizeof(W);
                        if (s1 >= inLo && s1 < inHi) cp_async<sizeof(W)>(dst + 16u * c + k * sizeof(W), s1);
                    }
                }
            }
        }
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        const uint32_t t = t0 + (uint32_t)s * G;
        if (t < nTiles) issue(t, sm0 + (uint32_t)s * sbytes);
        cp_async_commit();
    }
    const bool allSlots = p.V == NT * NREG;
    uint32_t k = 0;
    for (uint32_t t = t0; t < nTiles; t += G) {
        cp_async_wait<S - 2>();
        __syncthreads();
        {  // refill the stage read in the previous iteration
            const uint32_t tn = t + (uint32_t)(S - 1) * G;
            const uint32_t kn = (k + S - 1) % S;
            if (tn < nTiles) issue(tn, sm0 + kn * sbytes);
            cp_async_commit();
        }
        const TileBase<uint32_t> now = walk.seek(t);
        const uint32_t sb = sm0 + k * sbytes;
        // byte offset of the tile base inside its 16-byte chunk
        const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(in + now.in) & 15u);
        W* __restrict__ dst = opaque(out + now.out);
        uint32_t m;
        if constexpr (NREG == 16) {
            m = now.need == 0 ? (smask & 0xffffu) : now.need == 1 ? (smask >> 16)
                : now.need == 2 ? (smaskHi & 0xffffu) : (smaskHi >> 16);
        } else {
            m = (smask >> (now.need * NREG)) & ((1u << NREG) - 1u);
        }
        if (now.need == 0 && allSlots) {
#pragma unroll
            for (int r = 0; r < NREG; ++r) {
                const uint32_t a = sb + (spk[r] & 0xffffffu) + ((sh + (spk[r] >> 24)) & 15u);
                stg_(elem_addr(dst, gout[r]), lds<W>(a));
            }
        } else {
#pragma unroll
            for (int r = 0; r < NREG; ++r)
                if (m & (1u << r)) {
                    const uint32_t a = sb + (spk[r] & 0xffffffu) + ((sh + (spk[r] >> 24)) & 15u);
                    stg_(elem_addr(dst, gout[r]), lds<W>(a));
                }
        }
        k = (k + 1 == (uint32_t)S) ? 0u : k + 1;
    }
    cp_async_wait<0>();
}

// vector-gather tile: 4/8-byte words, 4/8/16 slots, 3 or 4 stages, 32-bit indices
const void* pick_tile_vg(int esize, int nreg, int stages) {
#define TT_PICKVG(W, S)                                                      \
    switch (nreg) {                                                          \
        case 4: return (const void*)&tile_vg_kernel<W, 4, S>;               \
        case 8: return (const void*)&tile_vg_kernel<W, 8, S>;               \
        case 16: return (const void*)&tile_vg_kernel<W, 16, S>;             \
        default: return nullptr;                                             \
    }
    if (esize == 4) {
        if (stages == 3) { TT_PICKVG(uint32_t, 3) }
        if (stages == 4) { TT_PICKVG(uint32_t, 4) }
    } else if (esize == 8) {
        if (stages == 3) { TT_PICKVG(uint64_t, 3) }
        if (stages == 4) { TT_PICKVG(uint64_t, 4) }
    }
    return nullptr;
#undef TT_PICKVG
}

}  // namespace tt
