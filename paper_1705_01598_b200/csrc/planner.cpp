// planner.cpp -- host planner: validate (row a-1), normalise/fuse (a-2),
// classify (a-3), choose parameters with the B200 model (a-4), materialise
// the kernel parameter block (a-5), describe.  No CUDA runtime calls here, so
// the planner runs on a machine without a GPU (tt_plan_offline).
//
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <vector>

#include "tt_internal.h"

namespace tt {

// --------------------------------------------------------------------------
// a-1 validate (P:L167 plan inputs; P:L82 h <= 32; R7-R11)
// --------------------------------------------------------------------------
tt_status_t validate(int rank, const int64_t* dims, const int* perm, size_t elem_size) {
    if (rank < 1 || rank > kMaxDims || dims == nullptr || perm == nullptr)
        return TT_INVALID_PARAMETER;
    bool seen[kMaxDims] = {};
    long double vol = 1;
    for (int i = 0; i < rank; ++i) {
        if (dims[i] < 1) return TT_INVALID_PARAMETER;
        if (perm[i] < 0 || perm[i] >= rank || seen[perm[i]]) return TT_INVALID_PARAMETER;
        seen[perm[i]] = true;
        vol *= (long double)dims[i];
    }
    if (elem_size != 4 && elem_size != 8) return TT_UNSUPPORTED;
    if (vol * (long double)elem_size >= (long double)(1LL << 62)) return TT_INVALID_PARAMETER;
    return TT_SUCCESS;
}

// --------------------------------------------------------------------------
// a-2 normalise: drop extent-1 dims (they never change a position, Eq. (1)
// P:L56 has a zero term for them) and fuse input dims i, i+1 that appear as
// ..., i, i+1, ... in the output order: both layouts then see them as one
// dimension of extent d[i]*d[i+1] (c(i+1,.) = c(i,.) * d(i) on both sides).
// --------------------------------------------------------------------------
static void fill_strides(Problem& pr) {
    int64_t acc = 1;
    for (int i = 0; i < pr.n; ++i) { pr.sin[i] = acc; acc *= pr.d[i]; }
    acc = 1;
    for (int j = 0; j < pr.n; ++j) { pr.sout[pr.p[j]] = acc; acc *= pr.d[pr.p[j]]; }
    pr.vol = acc;
    pr.span = acc;
}

Problem normalize(int rank, const int64_t* dims, const int* perm, int esize, bool fuse) {
    Problem pr;
    pr.esize = esize;
    if (!fuse) {
        pr.n = rank;
        for (int i = 0; i < rank; ++i) { pr.d[i] = dims[i]; pr.p[i] = perm[i]; }
        fill_strides(pr);
        return pr;
    }
    // drop extent-1 dims
    int newIdx[kMaxDims];
    int n1 = 0;
    int64_t d1[kMaxDims];
    for (int i = 0; i < rank; ++i) {
        if (dims[i] > 1) { newIdx[i] = n1; d1[n1++] = dims[i]; }
        else newIdx[i] = -1;
    }
    int p1[kMaxDims];
    int m = 0;
    for (int j = 0; j < rank; ++j)
        if (newIdx[perm[j]] >= 0) p1[m++] = newIdx[perm[j]];
    if (n1 == 0) {  // every extent is 1: a one-element copy
        pr.n = 1; pr.d[0] = 1; pr.p[0] = 0;
        fill_strides(pr);
        return pr;
    }
    // group output positions into runs of consecutive input dims
    int gStart[kMaxDims], gLen[kMaxDims], ng = 0;
    for (int j = 0; j < n1;) {
        int s = p1[j], len = 1;
        while (j + len < n1 && p1[j + len] == s + len) ++len;
        gStart[ng] = s; gLen[ng] = len; ++ng;
        j += len;
    }
    // groups sorted by input start give the fused input order
    int order[kMaxDims];
    for (int g = 0; g < ng; ++g) order[g] = g;
    std::sort(order, order + ng, [&](int x, int y) { return gStart[x] < gStart[y]; });
    int rankOf[kMaxDims];
    for (int r = 0; r < ng; ++r) {
        int g = order[r];
        rankOf[g] = r;
        int64_t e = 1;
        for (int k = 0; k < gLen[g]; ++k) e *= d1[gStart[g] + k];
        pr.d[r] = e;
    }
    pr.n = ng;
    for (int g = 0; g < ng; ++g) pr.p[g] = rankOf[g];  // groups are in output order
    fill_strides(pr);
    return pr;
}

// Strided problems (tt_plan_strided): the same Eq. (1) map between
// caller-given layouts, in[sum_i x_i s_in(i)] -> out[sum_j x_{p(j)} s_out(j)].
// Extent-1 dims are dropped; input dims i, i+1 that are consecutive in the
// output order are fused only when both layouts make them one dimension
// (s_in(i+1) = s_in(i) d_i and the same on the output side).
Problem normalize_strided(int rank, const int64_t* dims, const int* perm, int esize,
                          const int64_t* in_str, const int64_t* out_str, bool fuse) {
    Problem pr;
    pr.esize = esize;
    pr.dense = false;
    int64_t si[kMaxDims], so[kMaxDims];  // per input dim
    for (int i = 0; i < rank; ++i) si[i] = in_str[i];
    for (int j = 0; j < rank; ++j) so[perm[j]] = out_str[j];
    // keep dims with extent > 1, in output order
    int keep[kMaxDims], m = 0;
    for (int j = 0; j < rank; ++j)
        if (dims[perm[j]] > 1) keep[m++] = perm[j];
    if (m == 0) {
        pr.n = 1; pr.d[0] = 1; pr.p[0] = 0; pr.sin[0] = 1; pr.sout[0] = 1;
        pr.vol = 1; pr.span = 1;
        return pr;
    }
    // fuse output-order neighbours (a, b) with b = next input dim after a
    // among kept dims and contiguous strides on both sides
    int64_t gd[kMaxDims], gsi[kMaxDims], gso[kMaxDims];
    int gfirst[kMaxDims], ng = 0;
    for (int q = 0; q < m;) {
        const int a = keep[q];
        int64_t d = dims[a];
        int last = a, len = 1;
        while (fuse && q + len < m) {
            const int b = keep[q + len];
            bool nextIn = b > last;
            for (int i = last + 1; i < b && nextIn; ++i) nextIn = dims[i] == 1;
            if (!nextIn || si[b] != si[a] * d || so[b] != so[a] * d) break;
            d *= dims[b];
            last = b;
            ++len;
        }
        gd[ng] = d; gsi[ng] = si[a]; gso[ng] = so[a]; gfirst[ng] = a; ++ng;
        q += len;
    }
    // input order of the groups = ascending first input dim
    int order[kMaxDims];
    for (int g = 0; g < ng; ++g) order[g] = g;
    std::sort(order, order + ng, [&](int x, int y) { return gfirst[x] < gfirst[y]; });
    int rankOf[kMaxDims];
    for (int r = 0; r < ng; ++r) {
        const int g = order[r];
        rankOf[g] = r;
        pr.d[r] = gd[g];
        pr.sin[r] = gsi[g];
        pr.sout[r] = gso[g];
    }
    pr.n = ng;
    for (int g = 0; g < ng; ++g) pr.p[g] = rankOf[g];
    int64_t vol = 1, maxIn = 0, maxOut = 0;
    for (int i = 0; i < ng; ++i) {
        vol *= pr.d[i];
        maxIn += (pr.d[i] - 1) * pr.sin[i];
        maxOut += (pr.d[i] - 1) * pr.sout[i];
    }
    pr.vol = vol;
    pr.span = std::max(maxIn, maxOut) + 1;
    // the same layout as the dense problem of these dims: plan it as dense
    Problem dn = normalize(ng, pr.d, pr.p, esize, false);
    bool same = true;
    for (int i = 0; i < ng; ++i) same = same && dn.sin[i] == pr.sin[i] && dn.sout[i] == pr.sout[i];
    if (same) { dn.dense = true; return dn; }
    return pr;
}

// Element widening: when the fastest dim is unchanged (perm[0] == 0) every
// row of d0 elements is contiguous on both sides, so k consecutive elements
// can move as one (E*k)-byte word when k divides d0 (bit-exact: the words are
// opaque).  Returns k in {1, 2, 4} (E*k <= 16).
int widen_factor(const Problem& pr) {
    if (!pr.dense || pr.n < 2 || pr.p[0] != 0) return 1;
    const int kmax = 16 / pr.esize;
    for (int k = kmax; k >= 2; k /= 2)
        if (pr.d[0] % k == 0) return k;
    return 1;
}

Problem widen_problem(const Problem& pr, int k) {
    int64_t d[kMaxDims];
    for (int i = 0; i < pr.n; ++i) d[i] = pr.d[i];
    d[0] /= k;
    Problem w = normalize(pr.n, d, pr.p, pr.esize * k, true);  // d[0] may have become 1
    w.widen = pr.widen * k;
    return w;
}

// --------------------------------------------------------------------------
// a-4 model.  Constants are B200 measurements: the
// sustained copy bandwidth of MEASURED_PEAKS.json and per-tile / per-slot
// costs fitted from calibration sweeps (bench_suite.py --calibrate).
// --------------------------------------------------------------------------
namespace model {
constexpr double kBwBytesPerUs = 6.3e6;   // achievable streaming read+write (MEASURED_PEAKS hbm_gbs ~6.5e6)
constexpr double kSector = 32.0;          // L2 sector bytes (32-byte lines)
constexpr double kClockMHz = 1800.0;      // SM clock under a memory-bound load
constexpr double kIssuePerClk = 4.0;      // warp-instructions per SM per clock
constexpr double kTileInstr = 90.0;       // per warp per tile: Alg. 1 decode, barrier, loop
constexpr double kTileInstr64 = 160.0;    // same with 64-bit index arithmetic
constexpr double kSlotInstr = 11.0;       // per warp per slot: LDG, STS, LDS, STG, masks, address
constexpr double kSlotInstrSd = 9.0;      // same, slot-dim map (uniform slot strides)
constexpr double kLaunchUs = 3.0;         // launch + tail
constexpr double kRunBytes = 12.0;        // per contiguous run: DRAM burst/row locality overhead
constexpr double kInflightBytes = 49152;  // loads in flight per SM needed for full bandwidth
constexpr double kTileLatUs = 1.5;        // per tile iteration of one CTA: load latency + barrier
}  // namespace model

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Thresholds found by same-box A/B on the suites; the
// calibration sweeps that set them are in tools/ and profiles/round1_*.
namespace rule {
constexpr double kRowMinBytes = 512;      // row copy: rows of un-widened words (profiles/round1_ab_rowmin.txt)
constexpr double kRowMinBytesWide = 4096; // row copy: rows of widened words
constexpr double kRowMinBytes4 = 8192;    // row copy: un-widened 4-byte rows (round 2,
                                          // profiles/round2_ab_rowcopy_tile/)
constexpr double kT2dFill = 0.6;          // 2-D kernel: overall tile fill
constexpr double kT2dFillB4 = 0.9;        // 2-D kernel: output-side fill, 4-byte words (round1_ab_fillb.txt)
constexpr double kT2dFillB8 = 0.8;        // ... 8-byte words
constexpr int kSdRuleVmax = 8192;         // larger slot-dim tiles under the output-run rule (round1_knob_ab_sd_rule.txt)
}  // namespace rule

// Hacker's Delight unsigned division by invariant integers: l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1; the 33-bit sum umulhi(n, m) + n cannot
// overflow for n < 2^31.
void magic_u31(uint32_t d, uint32_t& m, uint32_t& l) {
    if (d == 0) d = 1;
    l = d <= 1 ? 0u : (uint32_t)(32 - __builtin_clz(d - 1));  // ceil(log2 d)
    m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
}

template <typename T>
static void fill_magic(T& t) {
    for (int g = 0; g < t.h; ++g) {
        if (t.gC[g] < (int64_t(1) << 31)) magic_u31((uint32_t)t.gC[g], t.gMC[g], t.gLC[g]);
        if (t.gD[g] < (int64_t(1) << 31)) magic_u31((uint32_t)t.gD[g], t.gMD[g], t.gLD[g]);
    }
}

// Expected sectors touched by a run of `bytes` starting at an address that is
// a multiple of `align` bytes (align a power of two).
static double run_sectors(double bytes, int64_t align) {
    if (align >= 32) return std::ceil(bytes / model::kSector);
    // start offset uniform over the multiples of align inside a sector
    // (bytes is a whole number: the sums below are exact in integers)
    const int64_t b = (int64_t)bytes;
    int64_t s = 0;
    int cnt = 0;
    for (int64_t off = 0; off < 32; off += align, ++cnt) s += (off + b + 31) >> 5;
    return (double)s / cnt;
}

static int64_t pow2_align(int64_t x) {  // largest power of two dividing x (x>0), capped
    if (x == 0) return 1 << 20;
    return std::min<int64_t>(x & -x, 1 << 20);
}

struct TileCand {
    TileParams tp{};
    int64_t runIn = 0, runOut = 0;   // contiguous run lengths (elements) inside a full tile
    int threads = 0, nreg = 0;
    double cost_us = 1e30;
    double dram_eff = 0;
    double secIn = 0, secOut = 0;    // modelled sectors per full tile (read / write)
    double inflight = 0;             // modelled load bytes in flight per SM
    int smem = 0;
    bool ok = false;
    // slot-dim launch shape (tile_sd_kernel) won the model: tp carries its
    // sd* fields, threads its CTA size
    bool sd = false;
    int sdq = 0, sdr = 0;
};

// Shared-memory wavefronts for one warp access of element positions pos[32].
// The staging layout is injective (padded strides >= dense ones), so the
// lanes of one access touch distinct positions: the wavefront count is the
// largest number of lanes on one bank (4-byte words), or on one bank pair
// per half-warp phase (8-byte words; 16-byte words use the same half-warp
// model, as the padding search was calibrated with it).
static int warp_wavefronts(const int* pos, int nlanes, int esize) {
    if (nlanes <= 0) return 0;
    if (esize == 4) {
        uint8_t cnt[32] = {};
        for (int l = 0; l < nlanes; ++l) ++cnt[pos[l] & 31];
        uint8_t worst = 0;
        for (int b = 0; b < 32; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
        return worst;
    }
    const int per = 16, banks = 16;        // half-warp phases, bank pairs
    int total = 0;
    for (int ph = 0; ph * per < nlanes; ++ph) {
        uint8_t cnt[16] = {};
        for (int l = ph * per; l < std::min(nlanes, ph * per + per); ++l) ++cnt[pos[l] & (banks - 1)];
        uint8_t worst = 0;
        for (int b = 0; b < 16; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
        total += worst;
    }
    return total;
}

// Bank-conflict cost of a staging layout (the paper's TPR_shmem "calculated
// at runtime using the element positions given by Equation (6)"),
// for both the staging store (input order) and the transposed read (output
// order), on a sample of warps (cf. the 10 samples of P:L244).  Element
// (c_i) sits at sum_i c_i * sm[i].  The sampled lanes' tile coordinates do
// not depend on the layout, so they are decoded once (SmemSample) and every
// candidate layout costs one dot product per lane.
struct SmemSample {
    int a = 0, nacc = 0;
    int maxVary = -1;        // highest tile dim whose coordinate varies inside a sampled access
    int av = 0;              // maxVary + 1: relative coordinates of higher dims are all zero
    std::vector<int> nl;     // lanes per distinct access pattern
    std::vector<int> wt;     // sampled accesses with that pattern
    std::vector<int> coord;  // [pattern][lane][tile dim + 1], relative to lane 0; the last
                             // entry is a layout-independent extra offset (elements)
};

// Adding the same offset to every lane's position permutes the banks, so an
// access's wavefront count depends only on the lanes' coordinates relative to
// lane 0: sampled accesses with equal relative patterns are merged (weighted).
static int no_extra(const int*) { return 0; }

template <typename Extra = int (*)(const int*)>
static SmemSample smem_sample(const TileParams& tp, int sides = 3, Extra extra = no_extra) {
    SmemSample s;
    s.a = tp.a;
    const int V = tp.V;
    const int nw = (V + 31) / 32;
    const int step = std::max(1, nw / 8);
    const int A = tp.a + 1;
    std::vector<int> cur(32 * A);
    for (int w = 0; w < nw; w += step) {
        const int nl = std::min(32, V - w * 32);
        for (int side = 0; side < 2; ++side) {  // 0: staging store (input order), 1: transposed read
            if (!(sides & (1 << side))) continue;
            int c0[kMaxDims + 1] = {};
            // lane 0's coordinates by division, the next lanes by an odometer
            // step in this side's order (same values as decoding each lane)
            int c[kMaxDims + 1] = {};
            {
                int kk = w * 32;
                for (int jj = 0; jj < tp.a; ++jj) {
                    const int t = side == 0 ? jj : tp.tOutOrder[jj];
                    c[t] = kk % tp.tExt[t];
                    kk /= tp.tExt[t];
                }
            }
            for (int l = 0; l < 32; ++l) {
                if (l > 0 && l < nl) {
                    for (int jj = 0; jj < tp.a; ++jj) {
                        const int t = side == 0 ? jj : tp.tOutOrder[jj];
                        if (++c[t] < tp.tExt[t]) break;
                        c[t] = 0;
                    }
                }
                if (l >= nl)
                    for (int i = 0; i < tp.a; ++i) c[i] = 0;
                c[tp.a] = l < nl ? extra(c) : 0;
                if (l == 0)
                    for (int i = 0; i < A; ++i) c0[i] = c[i];
                for (int i = 0; i < A; ++i) cur[l * A + i] = l < nl ? c[i] - c0[i] : 0;
            }
            bool merged = false;
            for (int q = 0; q < s.nacc && !merged; ++q) {
                if (s.nl[q] != nl) continue;
                if (std::equal(cur.begin(), cur.end(), s.coord.begin() + (size_t)q * 32 * A)) {
                    ++s.wt[q];
                    merged = true;
                }
            }
            for (int l = 0; l < 32; ++l)
                for (int i = 0; i < tp.a; ++i)
                    if (cur[l * A + i] != 0) s.maxVary = std::max(s.maxVary, i);
            if (!merged) {
                s.nl.push_back(nl);
                s.wt.push_back(1);
                s.coord.insert(s.coord.end(), cur.begin(), cur.end());
                ++s.nacc;
            }
        }
    }
    s.av = s.maxVary + 1;
    // heaviest accesses first: the candidate costs are sums of integers, so
    // the order changes no cost, but a losing candidate exceeds its bound
    // (smem_cost_at) sooner
    if (s.nacc > 1) {
        std::vector<int> ord(s.nacc);
        for (int q = 0; q < s.nacc; ++q) ord[q] = q;
        std::stable_sort(ord.begin(), ord.end(), [&](int u, int v) { return s.wt[u] > s.wt[v]; });
        SmemSample t = s;
        for (int q = 0; q < s.nacc; ++q) {
            t.nl[q] = s.nl[ord[q]];
            t.wt[q] = s.wt[ord[q]];
            std::copy(s.coord.begin() + (size_t)ord[q] * 32 * A, s.coord.begin() + (size_t)(ord[q] + 1) * 32 * A,
                      t.coord.begin() + (size_t)q * 32 * A);
        }
        return t;
    }
    return s;
}

static long smem_cost(const SmemSample& s, int esize, const int32_t* sm, long bound = -1) {
    long cost = 0;
    int pos[32];
    const int* c = s.coord.data();
    for (int q = 0; q < s.nacc; ++q) {
        if (bound >= 0 && cost >= bound) return cost;  // already no better than the incumbent
        for (int l = 0; l < 32; ++l, c += s.a + 1) {
            int sp = c[s.a];
            for (int i = 0; i < s.av; ++i) sp += c[i] * sm[i];
            pos[l] = sp + 4096;  // relative positions may be negative: keep the low bits' meaning
        }
        cost += (long)s.wt[q] * warp_wavefronts(pos, s.nl[q], esize);
    }
    return cost;
}

// The padding searches change one pad at a time.  Raising pad[i] by c adds
// c * prod(ext[i..j-1]) to every stride sm[j], j >= i, so every sampled
// lane's position is linear in c: pos = base + c * w.  smem_line fixes the
// other pads, smem_cost_at then costs a candidate with one multiply-add per
// lane (only the low 5 bits matter: bank = pos mod 32).
struct SmemLine {
    std::vector<int> base, w;  // [access][lane]
};
// Returns the period of the cost in the candidate pad: cand and cand + 32/g
// give every lane the same bank (g = the largest power of two dividing every
// w mod 32), so candidates past the first period can never improve on it.
static int smem_line(const SmemSample& s, const int32_t* sm0, const int64_t* coef, SmemLine& ln) {
    const size_t n = (size_t)s.nacc * 32;
    ln.base.resize(n);
    ln.w.resize(n);
    const int* c = s.coord.data();
    int orw = 0;
    for (size_t k = 0; k < n; ++k, c += s.a + 1) {
        int64_t b = c[s.a], w = 0;
        for (int i = 0; i < s.av; ++i) {
            b += (int64_t)c[i] * sm0[i];
            w += (int64_t)c[i] * coef[i];
        }
        ln.base[k] = (int)(b & 1023);
        ln.w[k] = (int)(w & 1023);
        orw |= (int)(w & 31);
    }
    if (orw == 0) return 1;
    return 32 / (orw & -orw);
}
static long smem_cost_at(const SmemSample& s, int esize, const SmemLine& ln, int cand, long bound) {
    long cost = 0;
    int pos[32];
    for (int q = 0; q < s.nacc; ++q) {
        if (bound >= 0 && cost >= bound) return cost;
        const int* b = &ln.base[(size_t)q * 32];
        const int* w = &ln.w[(size_t)q * 32];
        for (int l = 0; l < 32; ++l) pos[l] = b[l] + cand * w[l];
        cost += (long)s.wt[q] * warp_wavefronts(pos, s.nl[q], esize);
    }
    return cost;
}

// Slot-dim thread map for a chosen generic tile (kernels.cu tile_sd_kernel):
// per phase a slot dim outside that side's contiguous run (stride >= run, so
// a warp still moves along the run) and R slots along it (R | ext preferred);
// passes Q so that threads * Q * R covers the phase's thread space.  Picks
// the (Q, R) instantiation with the most CTAs (tiles in flight) per SM, then
// the best slot fill; false if none fills at least 60 % of its slots within
// the kernel's launch bound.
template <typename OccOf>
static bool build_sd(TileParams& tp, int esize, int64_t runIn, int64_t runOut, OccOf occOf,
                     int& threads, int& sdq, int& sdr, int& ctasPerSm) {
    struct Pick { int slot = -1, R = 0, C = 0; double eff = 0; };
    auto pick_slot = [&](int ph, int RM) {
        Pick best;
        for (int t = 0; t < tp.a; ++t) {
            // outside the phase's contiguous run, or inside it with >= 32
            // contiguous elements before it (a warp still covers 32 in a row)
            const int64_t stride = ph == 0 ? tp.tSin[t] : tp.tSout[t];
            const int64_t before = ph == 0 ? tp.tCin[t] : tp.tCout[t];
            if (stride < (ph == 0 ? runIn : runOut) && before < 32) continue;
            // slot fill ext / (C * RM) with C = ceil(ext / R) chunks: the
            // largest R (fewest chunks) is best, smaller R never beats it
            const int ext = tp.tExt[t];
            const int R = std::min(RM, ext);
            const int C = (ext + R - 1) / R;
            const double eff = (double)ext / ((double)C * RM);
            if (eff > best.eff + 1e-9) { best.slot = t; best.R = R; best.C = C; best.eff = eff; }
        }
        return best;
    };
    double bestFill = 0;
    Pick bL, bS;
    int64_t bUL = 0, bUS = 0, bQL = 0, bQS = 0;
    for (int cfg = 0; cfg < 3; ++cfg) {
        const int QM = cfg == 0 ? 2 : cfg == 1 ? 1 : 4;
        const int RM = cfg == 0 ? 8 : cfg == 1 ? 16 : 4;
        const Pick L = pick_slot(0, RM), S = pick_slot(1, RM);
        if (L.slot < 0 || S.slot < 0) continue;
        const int64_t UL = (int64_t)tp.V / tp.tExt[L.slot] * L.C;
        const int64_t US = (int64_t)tp.V / tp.tExt[S.slot] * S.C;
        int64_t NT = (std::max(UL, US) + QM - 1) / QM;
        NT = (NT + 31) / 32 * 32;
        if (NT < 64) NT = 64;
        if (NT > (esize >= 8 ? 384 : 512)) continue;  // kernels.cu launch bounds
        const int64_t QL = (UL + NT - 1) / NT, QS = (US + NT - 1) / NT;
        // slots issued vs elements moved (per phase); tiles in flight per SM
        // (CTAs per SM) decide, fill breaks ties
        const double fill = std::min((double)tp.V / ((double)NT * QL * L.R),
                                     (double)tp.V / ((double)NT * QS * S.R));
        const int per = occOf((int)NT, QM, RM);
        const double score = per + 0.5 * fill;
        if (fill >= 0.6 && per > 0 && score > bestFill + 1e-9) {
            ctasPerSm = per;
            bestFill = score;
            bL = L; bS = S; bUL = UL; bUS = US; bQL = QL; bQS = QS;
            threads = (int)NT;
            sdq = QM;
            sdr = RM;
        }
    }
    if (bestFill <= 0) return false;
    tp.sdSlot[0] = bL.slot; tp.sdR[0] = bL.R; tp.sdC[0] = bL.C;
    tp.sdU[0] = (int32_t)bUL; tp.sdQ[0] = (int32_t)bQL;
    tp.sdSlot[1] = bS.slot; tp.sdR[1] = bS.R; tp.sdC[1] = bS.C;
    tp.sdU[1] = (int32_t)bUS; tp.sdQ[1] = (int32_t)bQS;
    return true;
}

// Tile extents for candidate run targets (Tin, Tout) in elements: need[i]
// elements of input dim i (1 = a grid dim), and the split dim of each side.
static void tile_need(const Problem& pr, int64_t Tin, int64_t Tout, int64_t* need, int& inSplit,
                      int& outSplit) {
    const int n = pr.n;
    for (int i = 0; i < n; ++i) need[i] = 1;
    inSplit = -1;
    outSplit = -1;
    // input side: M_m = first input dims, last one possibly split
    {
        int64_t P = 1;
        for (int i = 0; i < n; ++i) {
            if (P * pr.d[i] >= Tin) {
                int64_t ch = std::min(pr.d[i], ceil_div(Tin, P));
                need[i] = std::max(need[i], ch);
                if (ch < pr.d[i]) inSplit = i;
                break;
            }
            need[i] = pr.d[i];
            P *= pr.d[i];
        }
    }
    // output side: M_k = first output dims
    {
        int64_t P = 1;
        for (int j = 0; j < n; ++j) {
            int i = pr.p[j];
            if (P * pr.d[i] >= Tout) {
                int64_t ch = std::min(pr.d[i], ceil_div(Tout, P));
                need[i] = std::max(need[i], ch);
                if (ch < pr.d[i]) outSplit = i;
                break;
            }
            need[i] = pr.d[i];
            P *= pr.d[i];
        }
    }
}

// DRAM side of the tile model for extents need[] (no parameter block): the
// contiguous runs inside a full tile, their sector counts at the runs'
// alignment, and the modelled bytes of the whole launch.  False when the
// tile cannot be built (too large, a split chunk over the kernel's 8-bit
// packing, staging over the shared-memory limit).  The searches use
// bytes / bandwidth + launch as a lower bound of a tile's cost.
struct TileDram {
    int32_t V = 0;
    int64_t runIn = 0, runOut = 0;
    int smem = 0;
    double secIn = 0, secOut = 0, dram_eff = 0, bytes = 0;
    double nTiles = 0;
};
static bool tile_dram(const Problem& pr, const int64_t* need, int Vlimit, const DeviceInfo& dev,
                      TileDram& t) {
    const int n = pr.n;
    int64_t V = 1;
    for (int i = 0; i < n; ++i)
        if (__builtin_mul_overflow(V, need[i], &V) || V > Vlimit) return false;
    t.V = (int32_t)V;
    t.nTiles = 1;
    for (int i = 0; i < n; ++i) {
        if (need[i] == 1) {
            t.nTiles *= (double)pr.d[i];
        } else if (need[i] < pr.d[i]) {
            if (need[i] > 256) return false;  // split chunk: 8-bit packing
            t.nTiles *= (double)ceil_div(pr.d[i], need[i]);
        }
    }
    {
        int64_t r = 1;
        for (int i = 0; i < n; ++i) {
            r *= need[i];
            if (need[i] < pr.d[i]) break;
        }
        t.runIn = std::min<int64_t>(r, t.V);
        r = 1;
        for (int j = 0; j < n; ++j) {
            int i = pr.p[j];
            r *= need[i];
            if (need[i] < pr.d[i]) break;
        }
        t.runOut = std::min<int64_t>(r, t.V);
    }
    // smem footprint with the worst-case padding (layout chosen for the winner)
    {
        int64_t words = t.V + t.V / 4 + 64;  // choose_smem's padding cap
        t.smem = (int)(2 * ((words + 3) / 4 * 4) * pr.esize);
        if (t.smem > dev.max_smem_per_block) return false;
    }
    const double E = pr.esize;
    // alignment of the runs' starts: strides of the tile dims outside the
    // run and of the grid dims (need 1, or a split dim's chunk stride)
    int64_t aIn = 256, aOut = 256;  // allocations are at least 256-byte aligned
    for (int i = 0; i < n; ++i) {
        const bool tileDim = need[i] > 1, gridDim = need[i] == 1 || need[i] < pr.d[i];
        if (tileDim && pr.sin[i] >= t.runIn) aIn = std::min(aIn, pow2_align(pr.sin[i] * pr.esize));
        if (tileDim && pr.sout[i] >= t.runOut) aOut = std::min(aOut, pow2_align(pr.sout[i] * pr.esize));
        if (gridDim) {
            aIn = std::min(aIn, pow2_align(need[i] * pr.sin[i] * pr.esize));
            aOut = std::min(aOut, pow2_align(need[i] * pr.sout[i] * pr.esize));
        }
    }
    aIn = std::max<int64_t>(aIn, pr.esize);
    aOut = std::max<int64_t>(aOut, pr.esize);
    t.secIn = run_sectors(t.runIn * E, aIn) * ((double)t.V / t.runIn);
    t.secOut = run_sectors(t.runOut * E, aOut) * ((double)t.V / t.runOut);
    // partial-sector reads of neighbouring runs usually hit in L2; partial
    // writes cost a read-modify-write -- weight them fully.
    const double usefulSec = 2.0 * t.V * E / model::kSector;
    const double modelSec = 0.5 * (t.secIn + t.V * E / model::kSector) + t.secOut +
                            ((double)t.V / t.runIn + (double)t.V / t.runOut) * model::kRunBytes /
                                model::kSector;
    t.dram_eff = usefulSec / modelSec;
    // DRAM bytes scale with the elements actually moved (ragged tiles move fewer)
    t.bytes = (double)pr.vol / t.V * modelSec * model::kSector;
    return true;
}
// A lower bound of build_tile_need's cost over every launch shape it may
// pick: memory time at full memory-level parallelism; issue time with the
// fewest instructions any shape issues (every element one slot of the
// cheaper slot-dim kind, one warp's per-tile overhead); the per-tile latency
// floor at the most CTAs per SM any shape reaches (estimate_occupancy: the
// shapes use >= V/16 threads and >= 4 V registers, the same staging bytes).
// The cost combines max + 0.25 * rest, nondecreasing in each term; the 1e-9
// margin keeps the bound below the rounded cost.
static double tile_cost_lb(const TileDram& t, int esize, const DeviceInfo& dev) {
    const double t_mem = t.bytes / model::kBwBytesPerUs;
    const double perTile = model::kTileInstr + t.V / 32.0 * model::kSlotInstrSd * (esize > 4 ? 1.25 : 1.0);
    const double t_issue = t.nTiles * perTile / model::kIssuePerClk / std::max(1, dev.num_sms) / model::kClockMHz;
    const double bySmem = (double)(dev.max_smem_per_sm / (t.smem + 1024));
    const double byThreads = dev.max_threads_per_sm / std::max(32.0, t.V / 16.0);
    const double byRegs = dev.regs_per_sm / (4.0 * t.V);
    const double occ = std::max(1.0, std::floor(std::min({32.0, bySmem, byThreads, byRegs})));
    const double t_lat = std::ceil(t.nTiles / ((double)dev.num_sms * occ)) * model::kTileLatUs;
    const double top = std::max({t_mem, t_issue, t_lat});
    return (top + 0.25 * (t_mem + t_issue + t_lat - top) + model::kLaunchUs) * (1.0 - 1e-9);
}

// Build the tile with extents need[] (from tile_need).
// `full`: the whole parameter block (the winner); otherwise only what the
// searches compare is valid (c.tp's arrays beyond the tile's a / h entries
// are left as they were -- the memo reuses one scratch candidate).
static void build_tile_need(TileCand& c, const Problem& pr, const int64_t* need, int inSplit,
                            int outSplit, int Vmax, const DeviceInfo& dev, int forceThreads,
                            int maxR, int forceR, int VmaxSd, bool full = true,
                            const TileDram* known = nullptr) {
    c.runIn = c.runOut = 0;
    c.threads = c.nreg = 0;
    c.cost_us = 1e30;
    c.dram_eff = c.secIn = c.secOut = c.inflight = 0;
    c.smem = 0;
    c.ok = false;
    c.sd = false;
    c.sdq = c.sdr = 0;
    const int n = pr.n;
    TileDram dr;
    if (known) dr = *known;
    else if (!tile_dram(pr, need, std::max(Vmax, VmaxSd), dev, dr)) return;

    TileParams& tp = c.tp;
    if (full) {
        std::memset(&tp, 0, sizeof(tp));
    } else {
        tp.nSplit = 0;
        for (int ph = 0; ph < 2; ++ph) tp.sdSlot[ph] = tp.sdR[ph] = tp.sdC[ph] = tp.sdU[ph] = tp.sdQ[ph] = 0;
    }
    tp.V = dr.V;
    // tile dims: need > 1, ascending input dim
    int tileOf[kMaxDims];
    tp.a = 0;
    for (int i = 0; i < n; ++i) {
        tileOf[i] = -1;
        if (need[i] > 1) {
            tileOf[i] = tp.a;
            tp.tExt[tp.a] = (int32_t)need[i];
            tp.tSin[tp.a] = pr.sin[i];
            tp.tSout[tp.a] = pr.sout[i];
            ++tp.a;
        }
    }
    {
        int32_t acc = 1;
        for (int t = 0; t < tp.a; ++t) { tp.tCin[t] = acc; acc *= tp.tExt[t]; }
        int jj = 0;
        acc = 1;
        for (int j = 0; j < n; ++j) {
            int t = tileOf[pr.p[j]];
            if (t < 0) continue;
            tp.tOutOrder[jj++] = t;
            tp.tCout[t] = acc;
            acc *= tp.tExt[t];
        }
    }
    // grid dims (M̄_mk plus chunk indices of split dims): split dims first,
    // then the rest in input order (one common order, R3)
    int gridDim_[kMaxDims], ng = 0;
    bool isSplit[kMaxDims] = {};
    for (int i = 0; i < n; ++i) isSplit[i] = need[i] > 1 && need[i] < pr.d[i];
    if (inSplit >= 0 && isSplit[inSplit]) gridDim_[ng++] = inSplit;
    if (outSplit >= 0 && outSplit != inSplit && isSplit[outSplit]) gridDim_[ng++] = outSplit;
    for (int i = 0; i < n; ++i) {
        if (need[i] == 1) gridDim_[ng++] = i;
        else if (isSplit[i] && i != inSplit && i != outSplit) gridDim_[ng++] = i;  // cannot happen
    }
    tp.h = ng;
    tp.nSplit = 0;
    int64_t acc = 1;
    for (int g = 0; g < ng; ++g) {
        int i = gridDim_[g];
        int64_t ext = ceil_div(pr.d[i], need[i]);
        tp.gC[g] = acc;
        tp.gD[g] = ext;
        tp.gSin[g] = need[i] * pr.sin[i];
        tp.gSout[g] = need[i] * pr.sout[i];
        acc *= ext;
        if (isSplit[i]) {
            int s = tp.nSplit++;
            tp.splitLane[s] = g;
            tp.splitChunk[s] = (int32_t)need[i];
            tp.splitExt[s] = pr.d[i];
            tp.splitTile[s] = tileOf[i];
            tp.splitTail[s] = (int32_t)(pr.d[i] - (ext - 1) * need[i]);
        }
    }
    tp.nTiles = acc;
    if (full) fill_magic(tp);  // the searches only compare costs; the winner is rebuilt in full
    c.runIn = dr.runIn;
    c.runOut = dr.runOut;
    c.smem = dr.smem;

    // model: DRAM sectors of full tiles + slot issue + per-tile overhead,
    // minimised over the launch shape (threads x slots, NT*NREG >= V)
    {
        const double E = pr.esize;
        c.dram_eff = dr.dram_eff;
        c.secIn = dr.secIn;
        c.secOut = dr.secOut;
        const double bytes = dr.bytes;
        // slots of ragged tiles are partly idle but still issued (issue cost
        // scales with the tiles launched)
        const bool idx64 = pr.span >= (int64_t(1) << 31);
        // cost of one launch shape: memory time at the loads in flight it
        // allows, issue time, per-tile latency floor
        auto shape_cost = [&](int T, int slots, int occ, double slotInstr, double& inflight) {
            inflight = (double)occ * T * slots * E;
            const double mlp = std::min(1.0, inflight / model::kInflightBytes);
            const double t_mem = bytes / (model::kBwBytesPerUs * mlp);
            const double warps = T / 32.0;
            const double perTile = warps * ((idx64 ? model::kTileInstr64 : model::kTileInstr) +
                                            slots * slotInstr * (E / 4.0 > 1 ? 1.25 : 1.0));
            const double t_issue = (double)tp.nTiles * perTile / model::kIssuePerClk /
                                   std::max(1, dev.num_sms) / model::kClockMHz;
            const double t_lat = std::ceil((double)tp.nTiles / ((double)dev.num_sms * occ)) * model::kTileLatUs;
            const double top = std::max(std::max(t_mem, t_issue), t_lat);
            return top + 0.25 * (t_mem + t_issue + t_lat - top) + model::kLaunchUs;
        };
        for (int R : {8, 16, 4, 2, 1}) {  // ties: 8 slots (more warps, smaller code)
            if (tp.V > Vmax) break;        // tile only for the slot-dim kernel
            if (pr.esize >= 16 && R > 4) continue;  // 16-byte words: <= 4 slots
            // 16 slots: 256-thread CTAs, 32-bit indices only (kernels.cu launch bounds)
            if (R == 16 && idx64) continue;
            if (R > maxR) continue;
            if (forceR && R != forceR) continue;
            int T = (int)ceil_div(tp.V, R);
            T = (int)ceil_div(T, 32) * 32;
            if (forceThreads) {
                if ((long)forceThreads * R < tp.V) continue;
                T = forceThreads;
            }
            if (T > (R >= 16 ? 256 : 512)) continue;  // kernels.cu launch bounds
            if (T < 64 && R > 1) continue;
            // memory-level parallelism: bytes of loads in flight per SM (the
            // B200 analogue of the paper's MWP/MLP terms); latency
            // floor: every tile iteration of a CTA waits for its loads and a
            // barrier however few of its slots are valid (ragged tiles)
            const OccQuery oq{TT_KERNEL_TILE, pr.esize, R, 1, T, c.smem, idx64, 0, 0};
            double inflight = 0;
            const double cost = shape_cost(T, R, estimate_occupancy(oq, dev), model::kSlotInstr, inflight);
            if (c.threads == 0 || cost < c.cost_us) {
                c.cost_us = cost;
                c.threads = T;
                c.nreg = R;
                c.inflight = inflight;
            }
        }
        // slot-dim launch shape: per-pass bases instead of per-element
        // tables, so more CTAs (tiles in flight) per SM and tiles up to
        // VmaxSd elements
        if (VmaxSd > 0 && !idx64 && !forceThreads && !forceR) {
            int thr = 0, q = 0, r = 0, per = 0;
            auto occOf = [&](int T, int qq, int rr) {
                const OccQuery qs{TT_KERNEL_TILE, pr.esize, qq * rr, 1, T, c.smem, false, 0, 0, 0, qq, rr};
                return estimate_occupancy(qs, dev);
            };
            // build_sd writes only the sd* fields of tp (kept if it wins)
            if (build_sd(tp, pr.esize, c.runIn, c.runOut, occOf, thr, q, r, per)) {
                double inflight = 0;
                const int slots = std::max(tp.sdQ[0] * tp.sdR[0], tp.sdQ[1] * tp.sdR[1]);
                const double cost = shape_cost(thr, slots, per, model::kSlotInstrSd, inflight);
                if (c.threads == 0 || cost < c.cost_us) {
                    c.cost_us = cost;
                    c.threads = thr;
                    c.nreg = q * r;
                    c.inflight = inflight;
                    c.sd = true;
                    c.sdq = q;
                    c.sdr = r;
                } else {
                    for (int ph = 0; ph < 2; ++ph)
                        tp.sdSlot[ph] = tp.sdR[ph] = tp.sdC[ph] = tp.sdU[ph] = tp.sdQ[ph] = 0;
                }
            }
        }
        if (c.threads == 0) return;
    }
    c.ok = true;
}

// Build the tile of candidate run targets (Tin, Tout) in elements.
static TileCand build_tile(const Problem& pr, int64_t Tin, int64_t Tout, int Vmax,
                           const DeviceInfo& dev, int forceThreads, int maxR = 16, int forceR = 0,
                           int VmaxSd = 0) {
    int64_t need[kMaxDims];
    int inSplit, outSplit;
    tile_need(pr, Tin, Tout, need, inSplit, outSplit);
    TileCand c;
    build_tile_need(c, pr, need, inSplit, outSplit, Vmax, dev, forceThreads, maxR, forceR, VmaxSd);
    return c;
}

// Many run-target pairs give the same tile (a dim is taken whole from one
// target up): the searches of choose_plan evaluate each distinct tile once,
// keep only what the searches compare (model cost, runs), and the winner is
// rebuilt in full at the end.  A memo may be shared by the plans of one
// problem (the fp64 ring rule re-plans it with other options).
struct TileSumm {
    bool ok = false;
    double cost = 1e30;
    int64_t runIn = 0, runOut = 0;
    int64_t Tin = 0, Tout = 0;   // run targets that built it
    int VmaxSd = 0;
};

struct TileMemo {
    Problem prob;
    bool bound = false;
    bool same_problem(const Problem& p) const {
        if (!bound || p.n != prob.n || p.esize != prob.esize || p.dense != prob.dense || p.span != prob.span)
            return false;
        for (int i = 0; i < p.n; ++i)
            if (p.d[i] != prob.d[i] || p.p[i] != prob.p[i] || p.sin[i] != prob.sin[i] || p.sout[i] != prob.sout[i])
                return false;
        return true;
    }
    // One entry per distinct tile (extents, split dims, launch limits): the
    // DRAM model (with the tile volume, checked against each query's limit)
    // and, per slot-dim limit VmaxSd asked for, the full summary once the
    // lower bound did not settle a query.
    struct Slot {
        int VmaxSd = -1;
        bool full = false;
        TileSumm sm;
    };
    struct Ent {
        bool buildable = false;
        TileDram dr;
        double lb = 0;  // tile_cost_lb (buildable entries)
        int64_t Tin = 0, Tout = 0;
        Slot slot[2];
    };
    std::vector<int64_t> keys;   // kMaxDims + 3 per entry
    std::vector<Ent> val;
    std::vector<int> table;      // open addressing over entry indices, -1 = empty
    int width = 0;

    static uint64_t hash(const int64_t* k, int n) {
        uint64_t h = 1469598103934665603ull;
        for (int i = 0; i < n; ++i) h = (h ^ (uint64_t)k[i]) * 1099511628211ull;
        return h ^ (h >> 29);
    }
    void bind(const Problem& p) {
        if (same_problem(p)) return;
        prob = p;
        bound = true;
        width = p.n + 3;
        keys.clear();
        val.clear();
        table.assign(1024, -1);
    }
    // The entry of the tile with extents need[] (derived from run targets
    // (Tin, Tout) by tile_need); the memo must be bound to p.
    int lookup(const Problem& p, const int64_t* need, int inSplit, int outSplit, int64_t Tin, int64_t Tout,
               int Vmax, const DeviceInfo& dev, int forceThreads, int maxR, int forceR) {
        int64_t k[kMaxDims + 3];
        std::memcpy(k, need, sizeof(int64_t) * p.n);
        k[p.n] = Vmax;
        k[p.n + 1] = (int64_t)(inSplit + 1) * 64 + (outSplit + 1);
        k[p.n + 2] = (int64_t)forceThreads * 4096 + maxR * 64 + forceR;
        const size_t mask = table.size() - 1;
        size_t h = hash(k, width) & mask;
        for (; table[h] >= 0; h = (h + 1) & mask) {
            const int64_t* y = &keys[(size_t)table[h] * width];
            if (std::memcmp(k, y, sizeof(int64_t) * width) == 0) return table[h];
        }
        Ent e;
        e.buildable = tile_dram(p, need, 1 << 30, dev, e.dr);  // volume limit: per query
        if (e.buildable) e.lb = tile_cost_lb(e.dr, p.esize, dev);
        e.Tin = Tin;
        e.Tout = Tout;
        const int idx = (int)val.size();
        table[h] = idx;
        keys.insert(keys.end(), k, k + width);
        val.push_back(e);
        if (val.size() * 2 > table.size()) {  // grow and rehash
            std::vector<int> t2(table.size() * 2, -1);
            const size_t m2 = t2.size() - 1;
            for (size_t i = 0; i < val.size(); ++i) {
                size_t g = hash(&keys[i * width], width) & m2;
                while (t2[g] >= 0) g = (g + 1) & m2;
                t2[g] = (int)i;
            }
            table.swap(t2);
        }
        return idx;
    }
    // The summary of entry e under slot-dim limit VmaxSd.  A tile whose cost
    // cannot go below `below` (its DRAM lower bound is already >= below) is
    // reported as not ok without running the launch-shape model: the
    // searches only replace their incumbent on a strictly lower cost, so
    // such a tile could not have won.
    TileSumm summary(Ent& e, const Problem& p, const int64_t* need, int inSplit, int outSplit, int Vmax,
                     const DeviceInfo& dev, int forceThreads, int maxR, int forceR, int VmaxSd,
                     double below) {
        TileSumm none;
        none.Tin = e.Tin;
        none.Tout = e.Tout;
        none.VmaxSd = VmaxSd;
        if (!e.buildable || e.dr.V > std::max(Vmax, VmaxSd)) return none;  // ok = false
        Slot* sl = e.slot[0].VmaxSd == VmaxSd ? &e.slot[0] : e.slot[1].VmaxSd == VmaxSd ? &e.slot[1] : nullptr;
        if (sl && sl->full) return sl->sm;
        if (e.lb >= below) return none;  // cannot win against the caller's incumbent
        if (!sl) {
            sl = e.slot[0].VmaxSd < 0 ? &e.slot[0] : &e.slot[1];
            sl->VmaxSd = VmaxSd;
        }
        thread_local TileCand c;  // scratch: summaries only
        build_tile_need(c, p, need, inSplit, outSplit, Vmax, dev, forceThreads, maxR, forceR, VmaxSd, false,
                        &e.dr);
        sl->full = true;
        sl->sm = none;
        sl->sm.ok = c.ok;
        sl->sm.cost = c.cost_us;
        sl->sm.runIn = c.runIn;
        sl->sm.runOut = c.runOut;
        return sl->sm;
    }
    TileSumm get(const Problem& p, int64_t Tin, int64_t Tout, int Vmax, const DeviceInfo& dev,
                 int forceThreads, int maxR, int forceR, int VmaxSd, double below = 1e300) {
        bind(p);
        int64_t need[kMaxDims];
        int inSplit, outSplit;
        tile_need(p, Tin, Tout, need, inSplit, outSplit);
        Ent& e = val[lookup(p, need, inSplit, outSplit, Tin, Tout, Vmax, dev, forceThreads, maxR, forceR)];
        return summary(e, p, need, inSplit, outSplit, Vmax, dev, forceThreads, maxR, forceR, VmaxSd, below);
    }
};

// Shared-memory layout: per-dimension padded strides sm[i] = sm[i-1]*ext[i-1]
// + pad[i] (the L x (L+1) padding of P:L123 generalised to every level of
// the tile), chosen by coordinate descent on the conflict model, then by
// footprint.  Footprint is capped so the 16-bit staging offsets fit.
static void choose_smem_search(TileParams& tp, int esize);

// The layout search is a pure function of the tile's extents, output order
// and word size: recent answers are kept per thread (the plans of one
// problem -- narrow, widened, the fp64 ring alternative -- often share a tile).
static void choose_smem(TileParams& tp, int esize) {
    struct Entry {
        std::vector<int32_t> key;
        int32_t sm[kMaxDims];
        int32_t sbuf;
    };
    thread_local std::vector<Entry> cache;
    std::vector<int32_t> key;
    key.reserve(2 * tp.a + 2);
    key.push_back(tp.a);
    key.push_back(esize);
    for (int i = 0; i < tp.a; ++i) key.push_back(tp.tExt[i]);
    for (int i = 0; i < tp.a; ++i) key.push_back(tp.tOutOrder[i]);
    for (const Entry& e : cache)
        if (e.key == key) {
            for (int i = 0; i < tp.a; ++i) tp.tSm[i] = e.sm[i];
            tp.sbuf = e.sbuf;
            return;
        }
    choose_smem_search(tp, esize);
    Entry e;
    e.key = key;
    for (int i = 0; i < tp.a; ++i) e.sm[i] = tp.tSm[i];
    e.sbuf = tp.sbuf;
    if (cache.size() >= 32) cache.erase(cache.begin());
    cache.push_back(e);
}

static void choose_smem_search(TileParams& tp, int esize) {
    const int a = tp.a;
    int32_t pad[kMaxDims] = {};
    int32_t sm[kMaxDims];
    auto strides = [&](const int32_t* pd, int32_t* out) -> int64_t {
        int64_t acc = 1;
        for (int i = 0; i < a; ++i) {
            acc += (i > 0 ? pd[i] : 0);
            out[i] = (int32_t)acc;
            acc *= tp.tExt[i];
        }
        // footprint: last element + 1
        int64_t last = 0;
        for (int i = 0; i < a; ++i) last += (int64_t)(tp.tExt[i] - 1) * out[i];
        return last + 1;
    };
    const int64_t limit = std::min<int64_t>((65536 / esize) - 8, tp.V + tp.V / 4 + 64);
    strides(pad, sm);
    const SmemSample sample = smem_sample(tp);
    long best = smem_cost(sample, esize, sm);
    const int ideal_per_warp = esize == 4 ? 2 : esize == 8 ? 4 : 8;  // store + read
    const int nw = (tp.V + 31) / 32;
    const long ideal = (long)((nw + std::max(1, nw / 8) - 1) / std::max(1, nw / 8)) * ideal_per_warp;
    // pad[i] moves the strides of dims >= i only: dims above the highest one
    // that varies inside a sampled access cannot change any cost
    const int hi = std::min(a - 1, sample.maxVary);
    SmemLine ln;
    // coordinate descent; a dim is re-searched only if another pad changed
    // since its last search (otherwise it would find the same answer)
    int changes = 0, seenAt[kMaxDims];
    for (int i = 0; i < a; ++i) seenAt[i] = -1;
    for (int pass = 0; pass < 2 && best > ideal; ++pass) {
        for (int i = 1; i <= hi && best > ideal; ++i) {
            if (seenAt[i] == changes) continue;
            int32_t keep = pad[i];
            int32_t bestPad = keep;
            pad[i] = 0;
            const int64_t foot0 = strides(pad, sm);
            int64_t coef[kMaxDims] = {}, footW = 0, acc = 1;
            for (int j = i; j < a; acc *= tp.tExt[j], ++j) {
                coef[j] = acc;
                footW += (tp.tExt[j] - 1) * acc;
            }
            const int period = smem_line(sample, sm, coef, ln);
            for (int c = 0; c < period; ++c) {
                if (foot0 + c * footW > limit) continue;
                const long cst = smem_cost_at(sample, esize, ln, c, best);
                if (cst < best) { best = cst; bestPad = c; }
            }
            pad[i] = bestPad;
            if (bestPad != keep) ++changes;
            seenAt[i] = changes;
        }
    }
    const int64_t foot = strides(pad, sm);
    for (int i = 0; i < a; ++i) tp.tSm[i] = sm[i];
    tp.sbuf = (int32_t)((foot + 3) / 4 * 4);
}

// Vector-gather layout (kernels_vg.cu tile_vg_kernel) of a chosen generic
// tile: the run dims (the tile's first dims that are dense in the input),
// a run slot of 16-byte chunks holding the 16-byte-aligned superset of a run
// (worst-case shift 16 - E bytes) plus 16 bytes for the folded shift, padded
// slot strides for the other tile dims (multiples of 16 bytes so every slot
// stays 16-byte aligned), chosen on the transposed read's bank-conflict cost
// (P:L225), and the tile-base ring behind the S staging buffers.  Launch
// shape: NT threads x NREG store slots cover the tile; every thread owns
// K <= 4 (run, chunk) load items.  False when the runs are shorter than
// `minRunBytes`, a run needs more than 255 chunks, or it does not fit.
static bool build_vg(TileParams& tp, const Problem& pr, int S, int maxSmem, int minRunBytes,
                     int& threads, int& nreg, int& smem) {
    const int E = pr.esize;
    if ((E != 4 && E != 8) || !pr.dense || pr.span >= (int64_t(1) << 31)) return false;
    const int VPC = 16 / E;
    int M = 0;
    int64_t L = 1;
    while (M < tp.a && tp.tSin[M] == L) L *= tp.tExt[M++];
    if (M == 0 || L * E < minRunBytes || M == tp.a) return false;  // M == a: a plain copy
    const int64_t nch = (L * E + 16 - E + 15) / 16;  // chunks at the worst shift
    if (nch > 255) return false;
    tp.vgM = M;
    tp.vgL = (int32_t)L;
    tp.vgLtail = (int32_t)L;
    tp.vgRunBit = 0;
    for (int s = 0; s < tp.nSplit; ++s)
        if (tp.splitTile[s] == M - 1 && tp.splitTail[s] != tp.splitChunk[s]) {
            tp.vgRunBit = 1 << s;
            tp.vgLtail = (int32_t)(L / tp.tExt[M - 1] * tp.splitTail[s]);
        }
    tp.vgNR = (int32_t)(tp.V / L);
    tp.vgNch = (int32_t)nch;
    tp.vgE = E;
    int64_t span = 0;
    for (int t = 0; t < tp.a; ++t) span += (int64_t)(tp.tExt[t] - 1) * tp.tSin[t];
    tp.vgSpanIn = span + 1;
    // slot strides: tile dims < M dense (the run), the rest padded
    int32_t pad[kMaxDims] = {};
    int32_t sm[kMaxDims];
    const int64_t pitch = (nch + 1) * VPC;  // elements
    auto strides = [&]() -> int64_t {
        int64_t acc = 1;
        for (int t = 0; t < tp.a; ++t) {
            if (t == M) acc = pitch;
            acc += pad[t];
            sm[t] = (int32_t)acc;
            acc *= tp.tExt[t];
        }
        int64_t last = 0;
        for (int t = M; t < tp.a; ++t) last += (int64_t)(tp.tExt[t] - 1) * sm[t];
        return last + pitch;
    };
    // the transposed read only; an element of run r sits q_r = (run offset
    // mod 16 bytes) further (the folded shift, kernels_vg.cu)
    auto qshift = [&](const int* c) {
        int64_t off = 0;
        for (int t = M; t < tp.a; ++t) off += (int64_t)c[t] * tp.tSin[t];
        return (int)(off % VPC);
    };
    const SmemSample sample = smem_sample(tp, 2, qshift);
    strides();
    long best = smem_cost(sample, E, sm);
    SmemLine ln;
    for (int pass = 0; pass < 2; ++pass)
        for (int t = M; t < tp.a; ++t) {
            int32_t bestPad = pad[t];
            pad[t] = 0;
            const int64_t foot0 = strides();
            int64_t coef[kMaxDims] = {}, footW = 0, acc = 1;
            for (int j = t; j < tp.a; acc *= tp.tExt[j], ++j) {
                coef[j] = acc;
                footW += (tp.tExt[j] - 1) * acc;
            }
            const int period = std::max(smem_line(sample, sm, coef, ln), VPC);
            for (int c = 0; c < period; c += VPC) {
                if ((foot0 + c * footW) * E > 65536 * 2) continue;
                const long cst = smem_cost_at(sample, E, ln, c, best);
                if (cst < best) { best = cst; bestPad = c; }
            }
            pad[t] = bestPad;
        }
    const int64_t foot = strides();
    for (int t = 0; t < tp.a; ++t) tp.tSm[t] = sm[t];
    tp.sbuf = (int32_t)((foot + VPC - 1) / VPC * VPC);
    tp.vgTab = S * tp.sbuf * E;
    tp.vgInBytes = pr.span * E;
    smem = tp.vgTab + 128 * 16 + 16 * S;   // tile-base ring, full/empty mbarriers
    if (smem > maxSmem || (int64_t)tp.sbuf * E >= (int64_t(1) << 18)) return false;
    // store phase: NT threads x NREG slots cover the tile; load items <= 4
    threads = 0;
    const int64_t items = (int64_t)tp.vgNR * nch;
    for (int R : {8, 16, 4}) {
        int T = (int)((tp.V + R - 1) / R);
        T = (T + 31) / 32 * 32;
        if (T < 64) T = 64;
        if (T > (R >= 16 ? 512 : 1024)) continue;  // kernels_vg.cu launch bounds
        const int64_t K = (items + T - 1) / T;
        if (K > 4) continue;
        threads = T;
        nreg = R;
        tp.vgK = K <= 2 ? 2 : (int32_t)K;  // kernels: 2, 3 or 4 items
        break;
    }
    return threads > 0;
}

// Vectorised 2-D tiled kernel (TT_KERNEL_TILED2D): A = input dim 0, B = p[0].
// Returns false if the problem is not of that class or the vector width
// would be 1.  TA = 16*VW, TB = 16*VW*R with (VW, R) = (4,1) | (2,2) for 4-byte
// and (2,1) for 8-byte words (kernels.cu instantiations).
// Instantiated tiles (kernels.cu pick_tiled2d): 4-byte VW=4: {64,128}^2;
// 4-byte VW=2: 32x64, 64x64; 8-byte VW=2: {32,64}^2.
static bool tiled2d_tile_ok(int esize, int vec, int ta, int tb) {
    if (vec == 1) {  // scalar kernel instantiations
        if (esize == 4) return (ta == 64 && tb == 64) || (ta == 128 && tb == 64) || (ta == 64 && tb == 128);
        return (ta == 64 && tb == 64) || (ta == 32 && tb == 64) || (ta == 64 && tb == 32);
    }
    if (esize == 4 && vec == 4) return (ta == 64 || ta == 128) && (tb == 64 || tb == 128);
    if (esize == 4 && vec == 2) return (ta == 32 || ta == 64) && tb == 64;
    if (esize == 8 && vec == 2) return (ta == 32 || ta == 64) && (tb == 32 || tb == 64);
    return false;
}

static bool build_tiled2d(const Problem& pr, Tiled2DParams& t, int& vec, int& ta, int& tb,
                          double& fill, int wantA, int wantB, int order, int vec2) {
    if (pr.n < 2 || pr.p[0] == 0) return false;
    const int B = pr.p[0];
    // the kernels index in[b*sInB + a] and out[a*sOutA + b]: unit strides
    // for A on the input side and for B on the output side
    if (pr.sin[0] != 1 || pr.sout[B] != 1) return false;
    const int64_t dA = pr.d[0], dB = pr.d[B];
    // vectors of v elements: every row start a multiple of v on both sides
    auto vec_ok = [&](int v) {
        if (dA % v || dB % v) return false;
        for (int i = 0; i < pr.n; ++i) {
            if (i != 0 && pr.sin[i] % v) return false;
            if (i != B && pr.sout[i] % v) return false;
        }
        return true;
    };
    vec = 0;
    if (pr.esize == 4) {
        if (vec_ok(4)) vec = 4;
        else if (vec_ok(2)) vec = 2;
    } else if (vec_ok(2)) {
        vec = 2;
    }
    // 2-element vectors vs the scalar kernel (option t2d_vec2: 1 = always
    // vectors when the extents allow them, -1 = always scalar, 0 = the rule).
    //
    // Defaults from the same-box A/B (tools/vec2_ab.py,
    // profiles/round1_vec2_ab.jsonl): for 4-byte words the scalar kernel beat
    // 8-byte vectors on every shape (+12-17 %); for 8-byte words 16-byte
    // vectors win on large 2-D extents (+17 %) but lose on ragged ~100-600
    // extents (-6-8 %), so they are kept only when 64x64 tiles are >= 95 %
    // full.
    {
        const double fill64 = (double)dA / (64.0 * ceil_div(dA, 64)) * (double)dB / (64.0 * ceil_div(dB, 64));
        if (pr.esize == 4 && vec == 2 && vec2 <= 0) vec = 0;
        if (pr.esize == 8 && vec == 2 && (vec2 < 0 || (vec2 == 0 && fill64 < 0.95))) vec = 0;
    }
    if (vec == 0) vec = 1;  // scalar 2-D kernel (padded staging)
    // default tiles from the B200 calibration sweep (tools/sweep.py t2d,
    // profiles/round1_sweep_t2d.md): 64 x 128 for 4-byte words with 16-byte
    // vectors, 64 x 64 otherwise; two CTAs per SM, B-chunks fastest.
    if (pr.esize == 4) { ta = 64; tb = vec == 4 ? 128 : 64; }
    else { ta = 64; tb = 64; }
    // scalar kernel: 64 x 64 (tools/sweep_t2d_async.py on odd-extent S2
    // shapes: fp64 64x64 at 4 CTAs/SM beat 32x64 at 3 by 8-18 %)
    if (vec == 1) { ta = 64; tb = 64; }
    if (wantA || wantB) {
        if (wantA) ta = wantA;
        if (wantB) tb = wantB;
        if (!tiled2d_tile_ok(pr.esize, vec, ta, tb)) return false;
    }
    std::memset(&t, 0, sizeof(t));
    t.nSplit = 2;
    t.splitLane[0] = 0;
    t.splitLane[1] = 1;
    t.splitChunk[0] = ta;
    t.splitChunk[1] = tb;
    const int64_t nA = ceil_div(dA, ta), nB = ceil_div(dB, tb);
    t.splitTail[0] = (int32_t)(dA - (nA - 1) * ta);
    t.splitTail[1] = (int32_t)(dB - (nB - 1) * tb);
    t.sInB = pr.sin[B];
    t.sOutA = pr.sout[0];
    int g = 0;
    int64_t acc = 1;
    auto add = [&](int64_t ext, int64_t sIn, int64_t sOut) {
        t.gC[g] = acc; t.gD[g] = ext; t.gSin[g] = sIn; t.gSout[g] = sOut;
        acc *= ext; ++g;
    };
    // Tile order: consecutive tiles run concurrently on neighbouring CTAs, so
    // the fastest grid dim decides which side's DRAM rows are streamed whole.
    // B-chunks fastest keeps whole OUTPUT rows in flight (writes are the
    // costlier side on B200, calibration sweep); A-fastest the input rows.
    if (order == 1) {
        add(nA, (int64_t)ta * pr.sin[0], (int64_t)ta * pr.sout[0]);
        add(nB, (int64_t)tb * pr.sin[B], (int64_t)tb * pr.sout[B]);
        t.splitLane[0] = 0;
        t.splitLane[1] = 1;
    } else {
        add(nB, (int64_t)tb * pr.sin[B], (int64_t)tb * pr.sout[B]);
        add(nA, (int64_t)ta * pr.sin[0], (int64_t)ta * pr.sout[0]);
        t.splitLane[0] = 1;
        t.splitLane[1] = 0;
    }
    for (int i = 1; i < pr.n; ++i)
        if (i != B) add(pr.d[i], pr.sin[i], pr.sout[i]);
    t.h = g;
    t.nTiles = acc;
    fill_magic(t);
    fill = (double)pr.vol / ((double)acc * ta * tb);
    return true;
}

// TMA-staged 2-D transpose (kernels_tma.cu): the Tiled class with every
// stride a multiple of 16 bytes (cuTensorMapEncodeTiled) and at most 3 batch
// dims (tensor rank <= 5).  Boxes: 64 x 64 (4-byte) / 32 x 64 (8-byte words).
static bool build_tma2d(const Problem& pr, Tma2DParams& t) {
    const int E = pr.esize;
    if ((E != 4 && E != 8) || pr.n < 2 || pr.n > 5 || pr.p[0] == 0) return false;
    const int B = pr.p[0];
    if (pr.sin[0] != 1 || pr.sout[B] != 1) return false;
    std::memset(&t, 0, sizeof(t));
    t.TA = E == 4 ? 64 : 32;
    t.TB = 64;
    t.nb = pr.n - 2;
    t.rank = pr.n;
    t.gDimIn[0] = pr.d[0];
    t.gDimIn[1] = pr.d[B];
    t.gDimOut[0] = pr.d[B];
    t.gDimOut[1] = pr.d[0];
    t.gStrideIn[0] = (uint64_t)pr.sin[B] * E;
    t.gStrideOut[0] = (uint64_t)pr.sout[0] * E;
    int k = 0;
    for (int i = 1; i < pr.n; ++i) {
        if (i == B) continue;
        t.bExt[k] = (int32_t)pr.d[i];
        t.gDimIn[2 + k] = pr.d[i];
        t.gDimOut[2 + k] = pr.d[i];
        t.gStrideIn[1 + k] = (uint64_t)pr.sin[i] * E;
        t.gStrideOut[1 + k] = (uint64_t)pr.sout[i] * E;
        ++k;
    }
    for (int r = 0; r < t.rank; ++r)
        if (t.gDimIn[r] >= (uint64_t(1) << 32) || t.gDimIn[r] == 0) return false;
    for (int r = 0; r + 1 < t.rank; ++r)
        if (t.gStrideIn[r] % 16 || t.gStrideOut[r] % 16 || t.gStrideIn[r] >= (uint64_t(1) << 40) ||
            t.gStrideOut[r] >= (uint64_t(1) << 40))
            return false;
    t.nA = (int32_t)ceil_div(pr.d[0], t.TA);
    t.nB = (int32_t)ceil_div(pr.d[B], t.TB);
    t.nTiles = (int64_t)t.nA * t.nB;
    for (int q = 0; q < t.nb; ++q) t.nTiles *= t.bExt[q];
    return t.nTiles < (int64_t(1) << 31);
}

int estimate_occupancy(const OccQuery& q, const DeviceInfo& dev) {
    // register counts of the tile kernels as compiled (ptxas -v, build/obj)
    int regs;
    if (q.kernel == TT_KERNEL_TILE && q.sdq) {
        regs = q.esize == 8 ? 80 : 64;
    } else if (q.kernel == TT_KERNEL_TILE) {
        const int r8 = q.esize == 8 ? 96 : 64;
        regs = q.nreg >= 16 ? 128 : q.nreg >= 8 ? r8 : q.nreg >= 4 ? 56 : q.nreg >= 2 ? 52 : 44;
        if (q.idx64) regs += 16;
    } else {
        regs = 64;
    }
    int byRegs = dev.regs_per_sm / std::max(1, regs * q.threads);
    int byThreads = dev.max_threads_per_sm / std::max(1, q.threads);
    int bySmem = q.smem > 0 ? dev.max_smem_per_sm / (q.smem + 1024) : 32;
    return std::max(1, std::min(std::min(byRegs, byThreads), std::min(bySmem, 32)));
}

// --------------------------------------------------------------------------
// a-3 classify + a-4 choose + a-5 materialise
// --------------------------------------------------------------------------
static tt_status_t choose_plan_m(Plan& plan, const DeviceInfo& dev, const tt_plan_options_t* opts,
                                 OccupancyFn occ, TileMemo* sharedMemo);

tt_status_t choose_plan(Plan& plan, const DeviceInfo& dev, const tt_plan_options_t* opts,
                        OccupancyFn occ) {
    return choose_plan_m(plan, dev, opts, occ, nullptr);
}

static tt_status_t choose_plan_m(Plan& plan, const DeviceInfo& dev, const tt_plan_options_t* opts,
                                 OccupancyFn occ, TileMemo* sharedMemo) {
    const Problem& pr = plan.prob;
    KernelChoice& kc = plan.kc;
    const int forced = opts ? opts->kernel : TT_KERNEL_AUTO;
    const int E = pr.esize;

    kc.idx64 = pr.span >= (int64_t(1) << 31);
    const bool acc = opts && opts->accumulate;
    if (acc && (kc.idx64 || E > 8 || (forced != TT_KERNEL_AUTO && forced != TT_KERNEL_TILE)))
        return TT_UNSUPPORTED;
    kc.acc = acc ? 1 : 0;

    // (i) rank 1 after fusion: copy (identity; "trivial" permutation)
    // (strided problems: the copy and row-copy kernels assume dense layouts)
    if (!acc && pr.n == 1 && pr.dense && (forced == TT_KERNEL_AUTO || forced == TT_KERNEL_COPY)) {
        kc.kernel = TT_KERNEL_COPY;
        kc.threads = opts && opts->threads ? opts->threads : 512;
        kc.vec = 16 / E;
        int perSm = opts && opts->ctas_per_sm ? opts->ctas_per_sm : 4;
        int64_t chunks = ceil_div(pr.vol * E, 16 * 4 * (int64_t)kc.threads);
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)dev.num_sms * perSm));
        kc.predicted_us = 2.0 * pr.vol * E / model::kBwBytesPerUs + model::kLaunchUs;
        kc.model_dram_eff = 1.0;
        return TT_SUCCESS;
    }
    if (forced == TT_KERNEL_COPY) return TT_UNSUPPORTED;

    // (ii) fastest dim unchanged with long rows: row copy, no staging
    const bool rowClass = pr.n >= 2 && pr.p[0] == 0 && pr.dense;
    // Minimum row bytes for the row copy.  Same-box A/B over the suites
    // (tools/ab_rowmin.sh, profiles/round1_ab_rowmin.txt): for widened rows
    // (several elements per word) the generic tile beat the row copy on 12
    // of 13 cases below 4 KB rows (up to 1.39x, one loss of 0.95x); for
    // un-widened rows it lost on 7 of 8, so those keep 512 B.
    // Round 2: un-widened 4-byte rows under 8 KB measured faster on the
    // generic tile (the tile-base ring and vector-gather kernels came after
    // the round-1 A/B; profiles/round2_ab_rowcopy_tile/).
    const double rowMin = pr.widen > 1 ? rule::kRowMinBytesWide
                          : (E == 4 ? rule::kRowMinBytes4 : rule::kRowMinBytes);
    if (forced == TT_KERNEL_ROWCOPY && !rowClass) return TT_UNSUPPORTED;
    if (!acc && rowClass && (forced == TT_KERNEL_ROWCOPY ||
                     (forced == TT_KERNEL_AUTO && pr.d[0] * E >= rowMin &&
                      !(opts && (opts->run_in || opts->run_out))))) {
        RowParams& r = plan.row;
        std::memset(&r, 0, sizeof(r));
        r.row = pr.d[0];
        r.nRows = pr.vol / pr.d[0];
        r.h = pr.n - 1;
        int64_t acc = 1;
        for (int j = 1; j < pr.n; ++j) {
            const int i = pr.p[j];
            r.rC[j - 1] = acc;
            r.rD[j - 1] = pr.d[i];
            r.rSin[j - 1] = pr.sin[i];
            acc *= pr.d[i];
            if (r.rC[j - 1] < (int64_t(1) << 31)) magic_u31((uint32_t)r.rC[j - 1], r.gMC[j - 1], r.gLC[j - 1]);
            if (r.rD[j - 1] < (int64_t(1) << 31)) magic_u31((uint32_t)r.rD[j - 1], r.gMD[j - 1], r.gLD[j - 1]);
        }
        kc.kernel = TT_KERNEL_ROWCOPY;
        kc.threads = opts && opts->threads ? opts->threads : 256;
        const int perSm = opts && opts->ctas_per_sm ? opts->ctas_per_sm : 4;
        // Few long rows (e.g. the sharded unpack's (inner, middle, P) rows of
        // megabytes): a warp per row leaves most warps idle, so cut each row
        // into nseg segments of `seg` elements (>= 2 KB, a multiple of 32
        // words; the last one may be shorter), about four per warp in all.
        // Segment k of row q is a virtual row v = q*nseg + k -- a new fastest
        // row dim of extent nseg and input stride seg.
        const int64_t warpsTotal = (int64_t)dev.num_sms * perSm * (kc.threads / 32);
        r.rowFull = r.row;
        r.seg = r.segTail = r.row;
        r.nseg = 1;
        if (r.nRows < 4 * warpsTotal && r.h < kMaxDims - 1) {
            const int64_t want = ceil_div(4 * warpsTotal, r.nRows);
            int64_t best = ceil_div(ceil_div(r.row, want), 32) * 32;
            best = std::max<int64_t>(best, ceil_div(2048, E));
            if (best < r.row) {
                const int64_t nseg = ceil_div(r.row, best);
                r.seg = best;
                r.segTail = r.row - (nseg - 1) * best;
                r.nseg = nseg;
                for (int j = r.h; j > 0; --j) {
                    r.rC[j] = r.rC[j - 1] * nseg;
                    r.rD[j] = r.rD[j - 1];
                    r.rSin[j] = r.rSin[j - 1];
                }
                r.rC[0] = 1;
                r.rD[0] = nseg;
                r.rSin[0] = best;
                r.h += 1;
                r.row = best;
                r.nRows *= nseg;
                for (int j = 0; j < r.h; ++j) {
                    if (r.rC[j] < (int64_t(1) << 31)) magic_u31((uint32_t)r.rC[j], r.gMC[j], r.gLC[j]);
                    if (r.rD[j] < (int64_t(1) << 31)) magic_u31((uint32_t)r.rD[j], r.gMD[j], r.gLD[j]);
                }
            }
        }
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)dev.num_sms * perSm,
                                                              ceil_div(r.nRows * 32, kc.threads)));
        kc.predicted_us = 2.0 * pr.vol * E / model::kBwBytesPerUs + model::kLaunchUs;
        kc.model_dram_eff = 1.0;
        return TT_SUCCESS;
    }
    if (forced == TT_KERNEL_ROWCOPY) return TT_UNSUPPORTED;
    if (forced != TT_KERNEL_AUTO && forced != TT_KERNEL_TILE && forced != TT_KERNEL_TILED2D)
        return TT_UNSUPPORTED;
    int vec2d = 0, ta2d = 0, tb2d = 0;
    double fill2d = 0;
    const bool force2d = forced == TT_KERNEL_TILED2D;
    const bool can2d = !acc && build_tiled2d(pr, plan.t2d, vec2d, ta2d, tb2d, fill2d,
                                     force2d && opts ? opts->run_in : 0,
                                     force2d && opts ? opts->run_out : 0,
                                     opts && opts->grid_order ? opts->grid_order : 2,
                                     opts ? opts->t2d_vec2 : 0);
    if (forced == TT_KERNEL_TILED2D && !can2d) return TT_UNSUPPORTED;
    // fill of the output-fastest (B) side alone: short B extents leave the
    // 2-D kernel short write runs and half-empty tiles
    // Same-box A/B over the S2/S3/Set-2 suites (tools/ab_fillb.sh,
    // profiles/round1_ab_fillb.txt): below these fills the generic tile won
    // (up to 1.5x); 8-byte words lost above 0.8.
    const double fillB2d = can2d ? (double)pr.d[pr.p[0]] / ((double)tb2d * ceil_div(pr.d[pr.p[0]], tb2d)) : 0.0;
    const double fillBMin = E == 4 ? rule::kT2dFillB4 : rule::kT2dFillB8;
    // Plans that end on the 2-D kernel (want2d below; TMA plans) keep the
    // generic tile only as the fallback for misaligned pointers: its launch
    // shape takes the estimated occupancy, so planning them does not load the
    // generic kernels' CUDA modules (the first plan of a process pays those).
    const bool want2dEarly = forced == TT_KERNEL_TILED2D ||
                             (forced == TT_KERNEL_AUTO && can2d && fill2d >= rule::kT2dFill &&
                              fillB2d >= fillBMin && !(opts && (opts->run_in || opts->run_out)));
    const OccupancyFn occG = (want2dEarly || (opts && opts->tma > 0)) ? nullptr : occ;

    // generic staged tile (Tiled / Packed / PackedSplit classes)
    // 512 threads x 8 slots, and staging byte offsets < 2^16 (16-bit packing)
    const int Vmax = std::min(4096, 57344 / E);
    // slot-dim map (tile_sd_kernel): 4-byte words and 8-byte words made of
    // two 4-byte elements by default (on fp64 tensors it measured mixed:
    // opt-in); larger tiles than the classic map (16 elements x 512 / 384
    // threads, 16-bit staging offsets)
    const int sdOpt = opts ? opts->slot_dims : 0;
    // the stages option belongs to the vector-gather kernel when that is requested
    const int stOpt = opts && opts->vector_gather <= 0 ? opts->stages : 0;
    const bool sdAllowed = sdOpt >= 0 && !acc && !kc.idx64 && !(stOpt >= 3 && sdOpt <= 0) &&
                           (E == 4 || (E == 8 && (sdOpt > 0 || pr.widen > 1))) &&
                           !(opts && (opts->threads || opts->slots));
    // The slot-dim shape inside the tile model (option sd_vmax > 0, tiles up
    // to 8192 elements) and whole-dimension run targets are off by default:
    // on the suites they won and lost by up to 2.4x case by case with equal
    // medians (tools/knob_sweep.sh); the model cannot rank them.  By default
    // the slot-dim map is applied after the classic tile choice, by real
    // occupancy (below), which measured no losses.
    const int sdVmaxReq = opts && opts->sd_vmax ? opts->sd_vmax : 0;
    const int VmaxSd = sdAllowed ? std::min<int>(E == 4 ? 8192 : 6144, sdVmaxReq) : 0;
    // Larger slot-dim tiles (up to 8192 elements) under the same output-run
    // rule as the prefix targets (rule::kSdRuleVmax, the tile
    // limit).  Same-box A/B on the suites (profiles/round1_knob_ab_sd_rule.txt):
    // 17 cases changed, median 1.016x, up to 1.28x, one loss of 0.88x; Set 2
    // median 0.796 -> 0.803 of memcpy.
    const int sdRule = rule::kSdRuleVmax;
    const int VmaxSdRule = (sdAllowed && VmaxSd == 0 && sdRule > 0) ? std::min(E == 4 ? 8192 : 6144, sdRule) : 0;
    std::vector<int64_t> targets;
    for (int64_t b : {64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384})
        targets.push_back(std::max<int64_t>(2, b / E));
    // Whole-dimension prefix products as run targets too (tiles without a
    // split dim, no ragged chunks).  They are searched separately: on the
    // suites (tools/knob_ab.sh, profiles/round1_knob_ab_prefix.txt) they won
    // up to 1.36x where they kept or lengthened the OUTPUT run and lost up to
    // 0.62x where they bought a longer input run with a shorter output run --
    // short write runs cost more on B200 than the sector model charges.  So a
    // prefix tile replaces the power-of-two choice only when the model prefers
    // it AND its output run is at least as long (and its input run not below
    // half, unless the output run at least doubles).
    std::vector<int64_t> prefix;
    {
        int64_t P = 1;
        for (int i = 0; i < pr.n && P * pr.d[i] <= std::max(Vmax, VmaxSd); ++i) {
            P *= pr.d[i];
            if (P >= 2) prefix.push_back(P);
        }
        P = 1;
        for (int j = 0; j < pr.n && P * pr.d[pr.p[j]] <= std::max(Vmax, VmaxSd); ++j) {
            P *= pr.d[pr.p[j]];
            if (P >= 2) prefix.push_back(P);
        }
        std::sort(prefix.begin(), prefix.end());
        prefix.erase(std::unique(prefix.begin(), prefix.end()), prefix.end());
    }
    TileSumm best;
    const int forceThreads = opts ? opts->threads : 0;
    const int forceR = opts ? opts->slots : 0;
    TileMemo localMemo;
    TileMemo& memo = sharedMemo ? *sharedMemo : localMemo;
    const bool runsForced = opts && (opts->run_in || opts->run_out);
    if (runsForced) {
        // forced run target(s): the other side still searches the targets
        for (int64_t ti : targets)
            for (int64_t to : targets) {
                const int64_t Tin = opts->run_in ? opts->run_in : ti;
                const int64_t Tout = opts->run_out ? opts->run_out : to;
                const TileSumm c = memo.get(pr, Tin, Tout, Vmax, dev, forceThreads, acc ? 8 : 16, forceR,
                                            VmaxSd, best.ok ? best.cost : 1e300);
                if (c.ok && (!best.ok || c.cost < best.cost)) best = c;
            }
    } else {
        // Three searches, each the first strictly cheapest tile over its pairs
        // of run targets in ascending order: S1 over targets^2, S2 over
        // (targets + prefix)^2, S3 (slot-dim tiles, VmaxSdRule) over (targets +
        // prefix + slot-dim prefix)^2.  The lists are sorted, so one pass over
        // the largest set visits each search's pairs in that search's order.
        std::vector<int64_t> sdPrefix;
        if (VmaxSdRule > 0) {
            for (int i = 0, P = 1; i < pr.n && P * pr.d[i] <= VmaxSdRule; ++i) {
                P *= (int)pr.d[i];
                if (P >= 2) sdPrefix.push_back(P);
            }
            for (int j = 0, P = 1; j < pr.n && P * pr.d[pr.p[j]] <= VmaxSdRule; ++j) {
                P *= (int)pr.d[pr.p[j]];
                if (P >= 2) sdPrefix.push_back(P);
            }
        }
        std::vector<int64_t> cand = targets;
        cand.insert(cand.end(), prefix.begin(), prefix.end());
        cand.insert(cand.end(), sdPrefix.begin(), sdPrefix.end());
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        const int nc = (int)cand.size();
        // per candidate: membership (bit 0: targets, bit 1: targets + prefix)
        // and the tile extents each side asks for (tile_need, one side each)
        std::vector<int> member(nc, 0);
        std::vector<int64_t> sideIn((size_t)nc * pr.n), sideOut((size_t)nc * pr.n);
        std::vector<int> splitIn(nc), splitOut(nc);
        for (int k = 0; k < nc; ++k) {
            const int64_t v = cand[k];
            if (std::binary_search(targets.begin(), targets.end(), v)) member[k] |= 3;
            if (std::binary_search(prefix.begin(), prefix.end(), v)) member[k] |= 2;
            // one side of tile_need each: need = the elementwise max of both
            int64_t P = 1;
            splitIn[k] = -1;
            for (int i = 0; i < pr.n; ++i) sideIn[(size_t)k * pr.n + i] = 1;
            for (int i = 0; i < pr.n; ++i) {
                if (P * pr.d[i] >= v) {
                    const int64_t ch = std::min(pr.d[i], ceil_div(v, P));
                    sideIn[(size_t)k * pr.n + i] = ch;
                    if (ch < pr.d[i]) splitIn[k] = i;
                    break;
                }
                sideIn[(size_t)k * pr.n + i] = pr.d[i];
                P *= pr.d[i];
            }
            P = 1;
            splitOut[k] = -1;
            for (int i = 0; i < pr.n; ++i) sideOut[(size_t)k * pr.n + i] = 1;
            for (int j = 0; j < pr.n; ++j) {
                const int i = pr.p[j];
                if (P * pr.d[i] >= v) {
                    const int64_t ch = std::min(pr.d[i], ceil_div(v, P));
                    sideOut[(size_t)k * pr.n + i] = ch;
                    if (ch < pr.d[i]) splitOut[k] = i;
                    break;
                }
                sideOut[(size_t)k * pr.n + i] = pr.d[i];
                P *= pr.d[i];
            }
        }
        memo.bind(pr);
        const bool s3 = VmaxSdRule > 0;
        // Pass 1: the distinct tiles of every search and, per search, the
        // first pair (in that search's order) giving each.  Pair index
        // x * nc + y follows every search's own order.
        std::vector<int> first[3];  // per memo entry: first pair index in S1 / S2 / S3, -1 = none
        std::vector<int> ents;      // distinct entries in order of appearance
        // Both sides' extents grow with the run target, so the tile volume is
        // nondecreasing along each row and column of pairs: past the largest
        // volume any search accepts, the rest of a row cannot be used.
        const double vAll = (double)std::max({Vmax, VmaxSd, s3 ? VmaxSdRule : 0});
        for (int x = 0; x < nc; ++x) {
            const int64_t* ni = &sideIn[(size_t)x * pr.n];
            for (int y = 0; y < nc; ++y) {
                const int m = member[x] & member[y];
                if (!m && !s3) continue;
                const int64_t* no = &sideOut[(size_t)y * pr.n];
                int64_t need[kMaxDims];
                double vol = 1;
                for (int i = 0; i < pr.n; ++i) {
                    need[i] = std::max(ni[i], no[i]);
                    vol *= (double)need[i];
                }
                if (vol > vAll) break;
                const int e = memo.lookup(pr, need, splitIn[x], splitOut[y], cand[x], cand[y], Vmax, dev,
                                          forceThreads, acc ? 8 : 16, forceR);
                if ((size_t)e >= first[0].size())
                    for (auto& f : first) f.resize(memo.val.size() + nc * nc, -1);
                const int pi = x * nc + y;
                if (first[0][e] < 0 && first[1][e] < 0 && first[2][e] < 0) ents.push_back(e);
                if ((m & 1) && first[0][e] < 0) first[0][e] = pi;
                if ((m & 2) && first[1][e] < 0) first[1][e] = pi;
                if (s3 && first[2][e] < 0) first[2][e] = pi;
            }
        }
        // Pass 2, per search: the tile with the lowest (cost, first pair) --
        // the first strictly cheapest in the search's order.  Tiles are
        // visited by ascending DRAM lower bound; once that bound exceeds the
        // incumbent's cost no later tile can win (cost >= bound), so only the
        // tiles that might are given the full launch-shape model.
        auto run = [&](int k, int vsd, TileSumm& b) {
            std::vector<std::pair<double, int>> order;  // (lower bound, entry)
            for (int e : ents)
                if (first[k][e] >= 0 && memo.val[e].buildable) order.push_back({memo.val[e].lb, e});
            std::sort(order.begin(), order.end(), [&](const std::pair<double, int>& u, const std::pair<double, int>& v) {
                return u.first < v.first || (u.first == v.first && first[k][u.second] < first[k][v.second]);
            });
            int bIdx = -1;
            for (const auto& o : order) {
                const int e = o.second, pi = first[k][e];
                if (b.ok && (o.first > b.cost || (o.first == b.cost && pi > bIdx))) break;
                const int x = pi / nc, y = pi % nc;
                int64_t need[kMaxDims];
                for (int i = 0; i < pr.n; ++i)
                    need[i] = std::max(sideIn[(size_t)x * pr.n + i], sideOut[(size_t)y * pr.n + i]);
                const TileSumm c = memo.summary(memo.val[e], pr, need, splitIn[x], splitOut[y], Vmax, dev,
                                                forceThreads, acc ? 8 : 16, forceR, vsd, 1e300);
                if (c.ok && (!b.ok || c.cost < b.cost || (c.cost == b.cost && pi < bIdx))) {
                    b = c;
                    bIdx = pi;
                }
            }
        };
        TileSumm b2, b3;
        run(0, VmaxSd, best);
        run(1, VmaxSd, b2);
        if (s3) run(2, VmaxSdRule, b3);
        if (!prefix.empty()) {
            const TileSumm& px = b2;
            const bool keepsOut = best.ok && px.ok && px.runOut >= best.runOut &&
                                  (2 * px.runIn >= best.runIn || px.runOut >= 2 * best.runOut);
            if (px.ok && (!best.ok || (px.cost < best.cost && keepsOut)))
                best = px;
        }
        if (s3 && best.ok) {
            const TileSumm& sx = b3;
            const bool keepsOut = sx.ok && sx.runOut >= best.runOut &&
                                  (2 * sx.runIn >= best.runIn || sx.runOut >= 2 * best.runOut);
            if (sx.ok && sx.cost < best.cost && keepsOut) best = sx;
        }
    }
    TileCand bestTile;
    if (best.ok)  // the winner in full
        bestTile = build_tile(pr, best.Tin, best.Tout, Vmax, dev, forceThreads, acc ? 8 : 16, forceR,
                              best.VmaxSd);
    if (!bestTile.ok) {
        // fall back to the smallest legal tile
        for (int64_t t = 64; t >= 2 && !bestTile.ok; t /= 2) {
            TileCand c = build_tile(pr, t, t, 12288, dev, forceThreads, acc ? 8 : 16);
            if (c.ok) bestTile = c;
        }
    }
    if (!bestTile.ok) return TT_INTERNAL_ERROR;
    const TileCand& bt = bestTile;

    plan.tile = bt.tp;
    if (!bt.sd) plan.tile.sdSlot[0] = plan.tile.sdSlot[1] = -1;
    choose_smem(plan.tile, E);
    kc.kernel = TT_KERNEL_TILE;
    kc.threads = bt.threads;
    kc.nreg = bt.nreg;
    // staging pipeline: register double buffer (default) or a cp.async ring
    // of 3 stages (32-bit indices only)
    kc.stages = (stOpt >= 3 && opts->slot_dims <= 0 && !kc.idx64 && !acc && !bt.sd) ? 3 : 0;
    // interleaved tiles (neighbouring tiles on concurrently running CTAs)
    // measured better than contiguous ranges on 72 of 84 suite cases
    plan.tile.interleave = (opts && opts->grid_order == 2) ? 0 : 1;
    kc.smem = (kc.stages ? kc.stages : 2) * plan.tile.sbuf * E;
    if (kc.smem > dev.max_smem_per_block) { kc.stages = 0; kc.smem = 2 * plan.tile.sbuf * E; }
    kc.vec = 1;
    kc.predicted_us = bt.cost_us;
    kc.model_dram_eff = bt.dram_eff;
    kc.m_runIn = bt.runIn;
    kc.m_runOut = bt.runOut;
    kc.m_secIn = bt.secIn;
    kc.m_secOut = bt.secOut;
    kc.m_inflight = bt.inflight;
    constexpr int kRing = 64 * 16;  // slot-dim kernels: tile-base ring behind the staging buffers
    auto occOf = [&](int T, int q, int r) {
        OccQuery qs{TT_KERNEL_TILE, E, q * r, 1, T, kc.smem + kRing, false, 0, 0, 0, q, r};
        int v = occG ? occG(qs, dev) : 0;
        return v > 0 ? v : estimate_occupancy(qs, dev);
    };
    if (bt.sd) {
        // the model picked the slot-dim launch shape (possibly a tile larger
        // than the classic map can hold)
        kc.sdq = bt.sdq;
        kc.sdr = bt.sdr;
        const int per = opts && opts->ctas_per_sm ? opts->ctas_per_sm
                                                  : occOf(kc.threads, kc.sdq, kc.sdr);
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tile.nTiles, (int64_t)dev.num_sms * per));
    }
    OccQuery q{TT_KERNEL_TILE, E, kc.nreg, kc.stages ? kc.stages : 1, kc.threads, kc.smem,
               kc.idx64, 0, 0, kc.acc};
    int perSm = opts && opts->ctas_per_sm ? opts->ctas_per_sm : (occG ? occG(q, dev) : 0);
    if (perSm <= 0) perSm = estimate_occupancy(q, dev);
    if (!bt.sd)
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tile.nTiles, (int64_t)dev.num_sms * perSm));
    // The model kept the classic map: switch to the slot-dim map anyway when
    // it keeps more tiles in flight per SM with the device's real occupancy
    // (measured on the suites: the win/loss boundary), or when forced.
    if (!bt.sd) {
        int thr = 0, sq = 0, sr = 0, perSd = 0;
        TileParams sdTile = plan.tile;
        if ((sdAllowed || (sdOpt > 0 && !acc && !kc.idx64 && (E == 4 || E == 8))) &&
            kc.stages == 0 && build_sd(sdTile, E, bt.runIn, bt.runOut, occOf, thr, sq, sr, perSd) &&
            (sdOpt > 0 || perSd > perSm)) {
            plan.tile = sdTile;
            kc.sdq = sq;
            kc.sdr = sr;
            kc.threads = thr;
            const int per = opts && opts->ctas_per_sm ? opts->ctas_per_sm : perSd;
            kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tile.nTiles, (int64_t)dev.num_sms * per));
        }
    }
    // slot-dim map with a cp.async ring of S stages (tile_sd_async_kernel):
    // S-1 tiles in flight per CTA without data registers.  Experimental,
    // options slot_dims > 0 with stages 3 or 4 (measured planning), or
    // off by default (suites: mixed, up to 1.18x faster
    // and 1.3x slower case by case, profiles/round1_ab_sd_async.txt).
    if (kc.sdq && !acc && !kc.idx64) {
        const int S = (opts && opts->slot_dims > 0 && stOpt >= 3) ? stOpt : 0;
        if ((S == 3 || S == 4) && (int64_t)S * plan.tile.sbuf * E + kRing <= dev.max_smem_per_block) {
            kc.stages = S;
            kc.smem = S * plan.tile.sbuf * E + kRing;
            OccQuery qa{TT_KERNEL_TILE, E, kc.sdq * kc.sdr, S, kc.threads, kc.smem, false, 0, 0, 0, kc.sdq, kc.sdr};
            int per = opts && opts->ctas_per_sm ? opts->ctas_per_sm : (occG ? occG(qa, dev) : 0);
            if (per <= 0)
                per = std::max(1, std::min({dev.max_smem_per_sm / (kc.smem + 1024),
                                            dev.max_threads_per_sm / kc.threads,
                                            dev.regs_per_sm / (kc.threads * 64)}));
            kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tile.nTiles, (int64_t)dev.num_sms * per));
        }
    }
    // vector-gather load phase (tile_vg_kernel): 16-byte cp.async chunks of
    // the aligned superset of every input run, S-stage ring
    // Default: fastest dimension unchanged after fusion (perm[0] == 0, rows
    // too short for the row copy) on 4-byte words or 8-byte words widened
    // from 4-byte pairs.  Same-box A/B (profiles/round2_ab_vg*.jsonl): on
    // those suite cases median 1.04x, up to 1.51x on the worst suite case
    // (5^12 fp32), losses down to 0.83x where the heuristic's output runs are
    // very long; on fp64 elements and on perm[0] != 0 gathers it lost.
    static const tt_plan_options_t zeroO{};
    const bool noOptsVg = opts == nullptr || std::memcmp(opts, &zeroO, sizeof(zeroO)) == 0;
    const int vgOpt = opts ? opts->vector_gather
                           : 0;
    const bool vgDefault = noOptsVg && pr.dense && pr.n >= 2 && pr.p[0] == 0 &&
                           (E == 4 || (E == 8 && pr.widen > 1));
    if ((vgOpt > 0 || vgDefault) && !acc && !kc.idx64) {
        TileParams vt = plan.tile;
        vt.sdSlot[0] = vt.sdSlot[1] = -1;
        const int S = opts && opts->stages >= 3 ? std::min(4, opts->stages) : 4;
        int thr = 0, nr = 0, sm = 0;
        vt.vgPolicy = opts ? opts->vg_policy : 0;
        if (build_vg(vt, pr, S, dev.max_smem_per_block, 32, thr, nr, sm)) {
            plan.tile = vt;
            kc.vg = 1;
            kc.sdq = kc.sdr = 0;
            kc.stages = S;
            kc.threads = thr;
            kc.nreg = nr;
            kc.smem = sm;
            OccQuery qv{TT_KERNEL_TILE, E, nr, S, thr, sm, false, 0, 0, 0, 0, 0, vt.vgK};
            int per = opts && opts->ctas_per_sm ? opts->ctas_per_sm : (occG ? occG(qv, dev) : 0);
            if (per <= 0)
                per = std::max(1, std::min({dev.max_smem_per_sm / (sm + 1024), dev.max_threads_per_sm / thr,
                                            dev.regs_per_sm / (thr * 64)}));
            kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tile.nTiles, (int64_t)dev.num_sms * per));
        }
    }
    // tile-base ring (kernels read the bases of their tiles from it): the
    // slot-dim kernels, and the classic register-pipeline kernel on 32-bit
    // indices (the classic cp.async variant and 64-bit plans decode in place)
    if (kc.kernel == TT_KERNEL_TILE && !kc.vg && (kc.sdq || (!kc.idx64 && kc.stages == 0))) {
        plan.tile.ringOff = (kc.stages >= 3 ? kc.stages : 2) * plan.tile.sbuf * E;
        kc.smem = plan.tile.ringOff + kRing;
    }
    kc.fb_threads = kc.threads;
    kc.fb_grid = kc.grid;
    kc.fb_smem = kc.smem;
    kc.fb_stages = kc.stages;

    // TMA-staged 2-D kernel (option tma): whole boxes through the Tensor
    // Memory Accelerator, ragged tiles clipped by the hardware
    if (opts && opts->tma > 0) {
        if (acc || !build_tma2d(pr, plan.tma)) return TT_UNSUPPORTED;
        kc.kernel = TT_KERNEL_TILED2D;
        kc.tma = 1;
        kc.vec = 1;
        kc.tile0 = plan.tma.TA;
        kc.tile1 = plan.tma.TB;
        kc.threads = 256;
        kc.stages = 3;
        kc.smem = 5 * plan.tma.TA * plan.tma.TB * E + 3 * 8 + 128;
        OccQuery qt{TT_KERNEL_TILED2D, E, 0, 1, 256, kc.smem, false, 0, 0, 0, 0, 0, 0};
        qt.tma = plan.tma.rank;
        int per = opts->ctas_per_sm ? opts->ctas_per_sm : (occ ? occ(qt, dev) : 0);
        if (per <= 0) per = std::max(1, dev.max_smem_per_sm / (kc.smem + 1024));
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.tma.nTiles, (int64_t)dev.num_sms * per));
        kc.predicted_us = 2.0 * pr.vol * E / model::kBwBytesPerUs + model::kLaunchUs;
        kc.model_dram_eff = 1.0;
        return TT_SUCCESS;
    }

    // Vectorised 2-D tiled kernel when the tiles are mostly full: it moves
    // VW elements per instruction on both sides (model: its issue cost is a
    // fraction of the generic kernel's, DRAM sectors are whole).
    const bool want2d = forced == TT_KERNEL_TILED2D ||
                        (forced == TT_KERNEL_AUTO && can2d && fill2d >= rule::kT2dFill &&
                         fillB2d >= fillBMin &&
                         !(opts && (opts->run_in || opts->run_out)));
    if (want2d) {
        kc.kernel = TT_KERNEL_TILED2D;
        kc.vec = vec2d;
        kc.tile0 = ta2d;
        kc.tile1 = tb2d;
        kc.threads = 256;
        // scalar 2-D kernel: register double buffer, or a cp.async ring of
        // 3-4 stages (tiled2d_sa_kernel; 32-bit indices)
        // Default: the ring (4 stages, 1 CTA/SM) for 8-byte words on a plain
        // rank-2 problem (no batch dims): +5-10 % over the register version
        // on large odd 2-D fp64 transposes; batched (rank >= 3) and 4-byte
        // cases stay on the register version (tools/sweep_t2d_async.py big,
        // profiles/round1_sweep_t2d_big.jsonl).
        // Suites: it lost where the output-fastest extent was short (585:
        // 0.87 -> 0.64 of memcpy, 154: -1 %), so only from 2048 up.
        const bool ringDefault = vec2d == 1 && E == 8 && pr.n == 2 && pr.d[pr.p[0]] >= 2048 &&
                                 !(opts && (opts->stages || opts->ctas_per_sm));
        const int st2 = opts && opts->stages >= 3 ? std::min(4, opts->stages) : (ringDefault ? 4 : 0);
        kc.stages = (vec2d == 1 && st2 && !kc.idx64) ? st2 : 0;
        kc.smem = vec2d == 1 ? (kc.stages ? kc.stages : 2) * ta2d * (tb2d + 1) * E
                             : 2 * ta2d * tb2d * E;
        OccQuery q2{TT_KERNEL_TILED2D, E, 0, vec2d, 256, kc.smem, kc.idx64, ta2d, tb2d, 0, kc.stages, 0};
        int occ2 = occ ? occ(q2, dev) : 0;
        if (occ2 <= 0) occ2 = std::min(8, dev.max_smem_per_sm / (kc.smem + 1024));
        // two CTAs per SM measured best (fewer concurrent tiles, whole DRAM
        // rows); never more than fit, so the persistent grid is one wave
        // (scalar kernel: 3 CTAs/SM for 4-byte words; 4 for 8-byte words --
        // beyond the 3 that fit, a second partial wave that balances the
        // tail, measured best)
        int per2 = opts && opts->ctas_per_sm ? opts->ctas_per_sm
                   : (ringDefault && kc.stages) ? 1
                   : vec2d == 1 ? (E == 8 ? 4 : std::min(3, occ2)) : std::min(2, occ2);
        kc.grid = (int)std::max<int64_t>(1, std::min<int64_t>(plan.t2d.nTiles, (int64_t)dev.num_sms * per2));
        const double bytes = 2.0 * pr.vol * E / std::max(0.3, std::min(1.0, fill2d + 0.3));
        kc.predicted_us = bytes / model::kBwBytesPerUs + model::kLaunchUs;
        kc.model_dram_eff = 1.0;
    }
    // 8-byte words on the generic tile (fp64, or fp32 pairs widened to 8
    // bytes): the slot-dim map with a 4-stage cp.async ring
    // (tile_sd_async_kernel) when that plan runs at one CTA per SM.  Same-box
    // A/B over the suites' 8-byte generic-tile cases
    // (profiles/round1_ab_sd_async8.txt): 18 of 20 faster, median 1.10x, none
    // slower; at 2+ CTAs per SM it was a wash; widened fp32 pairs 5 of 5
    // faster.  Planner-chosen plans only (no options).
    static const tt_plan_options_t zeroOpts{};
    const bool noOpts = opts == nullptr || std::memcmp(opts, &zeroOpts, sizeof(zeroOpts)) == 0;
    if (noOpts && E == 8 && pr.dense && kc.kernel == TT_KERNEL_TILE && !kc.idx64 && !acc && !kc.vg) {
        Plan alt;
        alt.device = plan.device;
        alt.stream = plan.stream;
        alt.rank = plan.rank;
        alt.prob = plan.prob;
        tt_plan_options_t o{};
        o.slot_dims = 1;
        o.stages = 4;
        if (choose_plan_m(alt, dev, &o, occ, &memo) == TT_SUCCESS && alt.kc.kernel == TT_KERNEL_TILE &&
            alt.kc.sdq && alt.kc.stages == 4) {
            OccQuery qa{TT_KERNEL_TILE, E, alt.kc.sdq * alt.kc.sdr, 4, alt.kc.threads, alt.kc.smem,
                        false, 0, 0, 0, alt.kc.sdq, alt.kc.sdr};
            int per = occ ? occ(qa, dev) : 0;
            if (per <= 0)
                per = std::max(1, std::min({dev.max_smem_per_sm / (alt.kc.smem + 1024),
                                            dev.max_threads_per_sm / alt.kc.threads,
                                            dev.regs_per_sm / (alt.kc.threads * 64)}));
            if (per == 1) {
                plan.tile = alt.tile;
                plan.kc = alt.kc;
            }
        }
    }

    return TT_SUCCESS;
}

// --------------------------------------------------------------------------
// describe (JSON)
// --------------------------------------------------------------------------
template <typename T>
static void arr(std::ostringstream& o, const T* v, int n) {
    o << "[";
    for (int i = 0; i < n; ++i) o << (i ? "," : "") << (long long)v[i];
    o << "]";
}

static const char* kernel_name(int k) {
    switch (k) {
        case TT_KERNEL_COPY: return "copy";
        case TT_KERNEL_TILE: return "tile";
        case TT_KERNEL_ROWCOPY: return "rowcopy";
        case TT_KERNEL_TILED2D: return "tiled2d";
        default: return "auto";
    }
}

std::string describe_json(const Plan& plan) {
    std::ostringstream o;
    const Problem& pr = plan.prob;
    const KernelChoice& kc = plan.kc;
    o << "{\"version\":" << TT_VERSION << ",\"device\":" << plan.device
      << ",\"rank\":" << plan.rank << ",\"dims\":";
    arr(o, plan.dims.data(), plan.rank);
    o << ",\"perm\":";
    arr(o, plan.perm.data(), plan.rank);
    o << ",\"elem_size\":" << pr.esize / plan.widen << ",\"word_size\":" << pr.esize
      << ",\"vol\":" << (long long)pr.vol;
    o << ",\"fused\":{\"rank\":" << pr.n << ",\"dims\":";
    arr(o, pr.d, pr.n);
    o << ",\"perm\":";
    arr(o, pr.p, pr.n);
    o << "},\"kernel\":\"" << kernel_name(kc.kernel) << "\",\"accumulate\":" << kc.acc
      << ",\"stages\":" << kc.stages
      << ",\"threads\":" << kc.threads
      << ",\"grid\":" << kc.grid << ",\"smem\":" << kc.smem << ",\"nreg\":" << kc.nreg
      << ",\"vec\":" << kc.vec << ",\"idx64\":" << (kc.idx64 ? "true" : "false")
      << ",\"launches\":1,\"plan_us\":" << plan.plan_us << ",\"predicted_us\":" << kc.predicted_us
      << ",\"model_dram_eff\":" << kc.model_dram_eff << ",\"widen\":" << plan.widen
      << ",\"dense\":" << (pr.dense ? "true" : "false") << ",\"span\":" << (long long)pr.span;
    if (kc.kernel == TT_KERNEL_TILE || kc.kernel == TT_KERNEL_TILED2D)
        o << ",\"model\":{\"run_in\":" << kc.m_runIn << ",\"run_out\":" << kc.m_runOut
          << ",\"sec_in\":" << kc.m_secIn << ",\"sec_out\":" << kc.m_secOut
          << ",\"inflight\":" << kc.m_inflight << "}";
    if (kc.kernel == TT_KERNEL_ROWCOPY) {
        const RowParams& r = plan.row;
        o << ",\"rowcopy\":{\"row\":" << (long long)r.row << ",\"nRows\":" << (long long)r.nRows
          << ",\"row_full\":" << (long long)r.rowFull << ",\"seg\":" << (long long)r.seg
          << ",\"seg_tail\":" << (long long)r.segTail << ",\"nseg\":" << (long long)r.nseg
          << ",\"row_c\":";
        arr(o, r.rC, r.h);
        o << ",\"row_d\":";
        arr(o, r.rD, r.h);
        o << ",\"row_sin\":";
        arr(o, r.rSin, r.h);
        o << "}";
    }
    if (plan.narrow) o << ",\"narrow\":" << describe_json(*plan.narrow);
    if (plan.measured)
        o << ",\"measured\":{\"candidates\":" << plan.n_candidates << ",\"best_ms\":"
          << plan.measured_ms << ",\"heuristic_ms\":" << plan.heuristic_ms << "}";
    if (kc.kernel == TT_KERNEL_TILED2D) {
        const Tiled2DParams& t = plan.t2d;
        o << ",\"tiled2d\":{\"TA\":" << kc.tile0 << ",\"TB\":" << kc.tile1 << ",\"nTiles\":"
          << (long long)t.nTiles << ",\"tails\":";
        arr(o, t.splitTail, 2);
        o << ",\"lanes\":";
        arr(o, t.splitLane, 2);
        o << ",\"sInB\":" << (long long)t.sInB << ",\"sOutA\":" << (long long)t.sOutA
          << ",\"grid_c\":";
        arr(o, t.gC, t.h);
        o << ",\"grid_d\":";
        arr(o, t.gD, t.h);
        o << ",\"grid_sin\":";
        arr(o, t.gSin, t.h);
        o << ",\"grid_sout\":";
        arr(o, t.gSout, t.h);
        o << "},\"tma\":" << kc.tma;
        if (kc.tma)
            o << ",\"tma_box\":{\"rank\":" << plan.tma.rank << ",\"TA\":" << plan.tma.TA << ",\"TB\":"
              << plan.tma.TB << ",\"nTiles\":" << (long long)plan.tma.nTiles << "}";
        o << ",\"fallback\":{\"kernel\":\"tile\",\"threads\":" << kc.fb_threads
          << ",\"grid\":" << kc.fb_grid << ",\"smem\":" << kc.fb_smem << ",\"nreg\":" << kc.nreg << "}";
    }
    if (kc.kernel == TT_KERNEL_TILE || kc.kernel == TT_KERNEL_TILED2D) {
        const TileParams& t = plan.tile;
        o << ",\"tile\":{\"V\":" << t.V << ",\"sbuf\":" << t.sbuf << ",\"nTiles\":"
          << (long long)t.nTiles
          << ",\"ext\":";
        arr(o, t.tExt, t.a);
        o << ",\"cin\":";
        arr(o, t.tCin, t.a);
        o << ",\"sm\":";
        arr(o, t.tSm, t.a);
        o << ",\"cout\":";
        arr(o, t.tCout, t.a);
        o << ",\"out_order\":";
        arr(o, t.tOutOrder, t.a);
        o << ",\"sin\":";
        arr(o, t.tSin, t.a);
        o << ",\"sout\":";
        arr(o, t.tSout, t.a);
        o << ",\"split_tile\":";
        arr(o, t.splitTile, t.nSplit);
        o << ",\"split_lane\":";
        arr(o, t.splitLane, t.nSplit);
        o << ",\"split_chunk\":";
        arr(o, t.splitChunk, t.nSplit);
        o << ",\"split_ext\":";
        arr(o, t.splitExt, t.nSplit);
        o << ",\"grid_c\":";
        arr(o, t.gC, t.h);
        o << ",\"grid_d\":";
        arr(o, t.gD, t.h);
        o << ",\"grid_sin\":";
        arr(o, t.gSin, t.h);
        o << ",\"grid_sout\":";
        arr(o, t.gSout, t.h);
        if (kc.vg)
            o << ",\"vg\":{\"M\":" << t.vgM << ",\"L\":" << t.vgL << ",\"Ltail\":" << t.vgLtail
              << ",\"runs\":" << t.vgNR << ",\"chunks\":" << t.vgNch << ",\"items\":" << t.vgK
              << ",\"stages\":" << kc.stages << "}";
        if (kc.sdq) {
            o << ",\"sd\":{\"q\":" << kc.sdq << ",\"r\":" << kc.sdr << ",\"slot\":";
            arr(o, t.sdSlot, 2);
            o << ",\"R\":";
            arr(o, t.sdR, 2);
            o << ",\"C\":";
            arr(o, t.sdC, 2);
            o << ",\"U\":";
            arr(o, t.sdU, 2);
            o << ",\"Q\":";
            arr(o, t.sdQ, 2);
            o << "}";
        }
        o << "}";
    }
    o << "}";
    return o.str();
}

}  // namespace tt
