// tt_internal.h -- plan representation shared by the host planner
// (planner.cpp, no CUDA runtime calls) and the launch layer (api.cu /
// kernels.cu).  Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
#pragma once

#include <cuda.h>  // CUtensorMap (the TMA 2-D kernel's parameter block)

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tt.h"

namespace tt {

constexpr int kMaxDims = TT_MAX_RANK;

// ---------------------------------------------------------------------------
// Normalised problem (row a-2): extent-1 dims dropped, in-order runs fused.
// dims[0] stride-1; output dim j is input dim perm[j].
// ---------------------------------------------------------------------------
struct Problem {
    int n = 0;
    int64_t d[kMaxDims] = {};
    int p[kMaxDims] = {};
    int esize = 4;
    int widen = 1;                // words are `widen` caller elements (planner.cpp widen_problem)
    bool dense = true;            // false: caller-given strides (tt_plan_strided)
    int64_t span = 1;             // 1 + the largest element offset on either side (index width)
    int64_t vol = 1;
    int64_t sin[kMaxDims] = {};   // c(i, I): input stride of input dim i
    int64_t sout[kMaxDims] = {};  // c(i, O): output stride of input dim i
};

// ---------------------------------------------------------------------------
// Generic staged-tile kernel parameters (Eqs. 2-6).
//
// A tile is the sub-volume M_mk (the union of the first input dims M_m and
// the first output dims M_k), with at most one split dim per side
// (PackedSplit).  Tile dims are listed in input order; the kernel
// reads a tile with input-order index k (Eq. 4), stages element (c_i) at
// shared position sum_i c_i * tSm[i] (Eq. 6 with padded strides tSm instead
// of the dense c(q_i, M_mk^I), chosen by the planner's bank-conflict model),
// and writes it with output-order index k' (Eq. 5).  The remaining dims (and the chunk
// index of split dims) are the "major" grid dims M̄_mk decoded per tile with
// the warp-parallel Algorithm 1 in ONE common order for both the
// read and the write base (reading R3).
// ---------------------------------------------------------------------------
struct TileParams {
    int64_t nTiles;
    int32_t V;          // tile volume (elements)
    int32_t sbuf;       // elements per shared-memory buffer incl. padding
    int32_t a;          // number of tile dims
    int32_t h;          // number of grid dims (<= 32, one warp lane each)
    int32_t nSplit;     // number of split tile dims (0..2)
    int32_t interleave; // 1: CTA b runs tiles b, b+G, ...; 0: a contiguous range per CTA
    int32_t betaZero;   // accumulate plans: beta == 0 (do not read out)
    double alpha, beta; // accumulate plans: out = alpha*perm(in) + beta*out (set per launch)
    int32_t splitLane[2];   // grid lane carrying the split dim's chunk index
    int32_t splitChunk[2];  // tile extent of the split dim
    int32_t splitTile[2];   // tile-dim index of the split dim
    int32_t splitTail[2];   // valid extent of the last chunk (== chunk if it divides)
    int64_t splitExt[2];    // full extent of the split dim
    // tile dims (tile-input order, i.e. ascending input dimension)
    int32_t tExt[kMaxDims];       // tile extent
    int32_t tCin[kMaxDims];       // c(q_i, M_mk^I): cumulative volume, tile-input order
    int32_t tSm[kMaxDims];        // staging (shared memory) stride, elements: tCin + padding
    int32_t tCout[kMaxDims];      // c(q_i, M_mk^O): cumulative volume, tile-output order
    int32_t tOutOrder[kMaxDims];  // tile dims in output order (indices into the above)
    int64_t tSin[kMaxDims];       // c(q_i, I): global input stride
    int64_t tSout[kMaxDims];      // c(q_i, O): global output stride
    // grid dims, one per warp lane (Alg. 1): b -> mod(floor(b / gC), gD) * stride
    int64_t gC[kMaxDims];
    int64_t gD[kMaxDims];
    int64_t gSin[kMaxDims];
    int64_t gSout[kMaxDims];
    // 32-bit multiply-shift division magic for / gC and / gD (see fast_div)
    uint32_t gMC[kMaxDims], gLC[kMaxDims], gMD[kMaxDims], gLD[kMaxDims];
    // slot-dim variant (tile_sd_kernel), per phase ph = 0 (load, tile-input
    // order) and 1 (store, tile-output order): every thread owns sdR
    // consecutive elements along tile dim sdSlot per pass, so the per-slot
    // offsets are uniform strides and only a per-pass base stays per thread.
    int32_t sdSlot[2];  // tile dim carrying the slots (-1: variant not used)
    int32_t sdR[2];     // slots per pass along it
    int32_t sdC[2];     // chunks of the slot dim, ceil(ext / sdR)
    int32_t sdU[2];     // thread-space size: V / ext * chunks
    int32_t sdQ[2];     // passes, ceil(sdU / threads)
    int32_t ringOff;    // slot-dim kernels: byte offset of the 64-entry tile-base ring in dynamic smem
    // vector-gather variant (tile_vg_kernel, kernels_vg.cu): the load phase
    // copies the 16-byte-aligned superset of every input run (the tile's
    // first vgM dims, contiguous in the input) in 16-byte cp.async chunks.
    // Run r of a tile sits in shared memory at a 16-byte-aligned slot; its
    // elements are shifted by the run start's offset inside its 16-byte chunk.
    int32_t vgM;        // run dims: tile dims 0 .. vgM-1 (tile-input order)
    int32_t vgL;        // run length (elements) of a full run
    int32_t vgLtail;    // run length when the run's split dim is at its ragged tail
    int32_t vgRunBit;   // need bit (1 or 2) of that split dim; 0 if the run is never ragged
    int32_t vgNR;       // runs per tile
    int32_t vgNch;      // 16-byte chunks per run slot at the worst-case shift
    int32_t vgK;        // load items (run, chunk) per thread
    int32_t vgE;        // word bytes
    int32_t vgTab;      // byte offset of the tile-base ring (128 x uint4) + mbarriers in dynamic smem
    int32_t vgPolicy;   // cache flavour of the chunk copies (kernels_vg.cu cp_async16_pred)
    int64_t vgSpanIn;   // largest input offset inside a tile + 1 (elements)
    int64_t vgInBytes;  // bytes of the input tensor (chunks are clipped to [in, in + vgInBytes))
};

// Row-copy (fastest dim unchanged, long rows; TiledCopy class P:L141): each
// row of `row` contiguous elements is contiguous on both sides.  Rows are
// enumerated in OUTPUT order over the remaining dims.
struct RowParams {
    int64_t row;        // elements per (virtual) row; = seg when rows are segmented
    int64_t nRows;      // virtual rows (segments x rows)
    // Segmented rows (few long rows): digit 0 of the row odometer is the
    // segment index (extent nseg, input stride seg); segment k of a row is
    // [k*seg, min((k+1)*seg, rowFull)), the last one segTail long.  Output
    // row r starts at (r / nseg) * rowFull + (r % nseg) * seg.
    int64_t rowFull;    // elements of a whole row (fused dim 0)
    int64_t seg, segTail;
    int64_t nseg;       // 1: not segmented
    int32_t h;          // remaining dims (output dims 1..n-1, output order)
    int64_t rC[kMaxDims];     // cumulative row count in output order
    int64_t rD[kMaxDims];     // extent
    int64_t rSin[kMaxDims];   // input stride
    uint32_t gMC[kMaxDims], gLC[kMaxDims], gMD[kMaxDims], gLD[kMaxDims];  // fast_div magic
};

// Two-dimensional vectorised tiled transpose (Tiled class): the
// fused problem's input dim A = 0 (stride 1) and the output-fastest input
// dim B = perm[0] form TA x TB tiles; every other dim is a batch dim.  Each
// thread moves VW x VW micro-tiles with VW-element vector accesses on both
// sides (register transpose + XOR-swizzled shared memory), which needs
// d[A] % VW == 0, d[B] % VW == 0 and VW*E-aligned pointers.  The grid
// fields mirror TileParams (lane 0 = chunk index along A, lane 1 along B,
// then batch dims), decoded by the same Algorithm-1 routine.
struct Tiled2DParams {
    int64_t nTiles;
    int32_t h;
    int32_t nSplit;          // always 2 (A and B)
    int32_t splitLane[2];    // 0, 1
    int32_t splitChunk[2];   // TA, TB
    int32_t splitTail[2];    // valid extent of the last chunk along A / B
    int64_t sInB;            // input stride of dim B (elements)
    int64_t sOutA;           // output stride of dim A (elements)
    int64_t gC[kMaxDims], gD[kMaxDims], gSin[kMaxDims], gSout[kMaxDims];
    uint32_t gMC[kMaxDims], gLC[kMaxDims], gMD[kMaxDims], gLD[kMaxDims];
};

// TMA-staged 2-D tiled transpose (kernels_tma.cu): tensor maps of the input
// (dims A, B, batch...) and the output (B, A, batch...), encoded per device
// pointer pair at launch (they hold the global address), tile grid.
struct alignas(64) Tma2DParams {
    CUtensorMap inMap, outMap;
    int64_t nTiles;
    int32_t nA, nB;        // chunks along A and B
    int32_t nb;            // batch dims (0..3)
    int32_t TA, TB;        // box extents along A and B
    int32_t rank;          // tensor rank 2 + nb
    int32_t bExt[3];
    // host-side geometry for encoding (elements; strides in bytes)
    uint64_t gDimIn[5], gDimOut[5], gStrideIn[4], gStrideOut[4];
};

struct KernelChoice {
    int kernel = TT_KERNEL_AUTO;   // tt_kernel_t
    int threads = 0;
    int nreg = 0;                  // slots per thread (TILE)
    int vec = 1;                   // elements per vector access
    int grid = 0;
    int smem = 0;                  // dynamic shared memory bytes
    bool idx64 = false;
    int tile0 = 0, tile1 = 0;      // TILED2D tile
    int fb_threads = 0, fb_grid = 0, fb_smem = 0;  // generic-tile fallback launch
    int fb_stages = 0;                               // its pipeline stages (the 2-D choice reuses `stages`)
    int stages = 0;                // generic tile: 0 = register double buffer, >= 3 = cp.async ring
    int acc = 0;                   // accumulate plan (f-3): generic tile with alpha/beta
    int sdq = 0, sdr = 0;          // generic tile, slot-dim variant: passes x slots (0 = classic)
    int vg = 0;                    // generic tile, vector-gather variant (tile_vg_kernel)
    int tma = 0;                   // TILED2D staged by TMA (tiled2d_tma_kernel)
    double predicted_us = 0.0;
    double model_dram_eff = 0.0;   // algorithmic / modelled DRAM bytes
    // model features of the generic tile (describe "model"; calibration)
    long long m_runIn = 0, m_runOut = 0;
    double m_secIn = 0, m_secOut = 0, m_inflight = 0;
};

struct DeviceInfo {
    int device = -1;               // -1: offline plan
    int num_sms = 148;
    int max_smem_per_block = 232448;
    int max_smem_per_sm = 233472;
    int max_threads_per_sm = 2048;
    int regs_per_sm = 65536;
};

// Occupancy oracle: CTAs per SM for a kernel configuration (launch layer
// supplies the CUDA answer; offline plans use an estimate).
struct OccQuery {
    int kernel, esize, nreg, vec, threads, smem;
    bool idx64;
    int ta, tb;  // TILED2D tile
    int acc;     // TILE accumulate variant
    int sdq, sdr;  // TILE slot-dim variant (passes, slots); 0 = classic; TILED2D: sdq = cp.async stages
    int vg;        // TILE vector-gather variant (nreg = slots, vec = stages)
    int tma;       // TILED2D TMA variant: tensor rank (0 = not TMA)
};
typedef int (*OccupancyFn)(const OccQuery&, const DeviceInfo&);

struct ShardInfo;  // defined in dist.cu
struct HostPipe;   // defined in api.cu (pipelined tt_execute_host)

struct Plan {
    int device = -1;
    void* stream = nullptr;
    int rank = 0;
    std::vector<int64_t> dims;     // as given
    std::vector<int> perm;
    Problem prob;                  // fused
    KernelChoice kc;
    TileParams tile{};
    RowParams row{};
    Tiled2DParams t2d{};
    Tma2DParams tma{};             // kc.tma plans
    struct TmaCache {              // tensor maps of the last (in, out) pair, per plan
        std::mutex mu;
        const void* in = nullptr;
        void* out = nullptr;
        CUtensorMap inMap, outMap;
    };
    TmaCache* tmaCache = nullptr;
    ShardInfo* shard = nullptr;    // sharded plans only
    bool measured = false;         // chosen by tt_plan_measure
    float measured_ms = 0.f, heuristic_ms = 0.f;
    int n_candidates = 0;
    double plan_us = 0.0;          // host time of the planning that built this plan (0: cache hit / clone)
    int widen = 1;                 // words of the fused problem = widen original elements
    Plan* narrow = nullptr;        // un-widened plan, for pointers not aligned to E*widen
    HostPipe* pipe = nullptr;      // lazily built by tt_execute_host
    ~Plan();
};

// planner.cpp ---------------------------------------------------------------
// Magic (m, l) such that floor(n / d) == (umulhi(n, m) + n) >> l for all
// 0 <= n < 2^31 and 1 <= d < 2^31.
void magic_u31(uint32_t d, uint32_t& m, uint32_t& l);
tt_status_t validate(int rank, const int64_t* dims, const int* perm, size_t elem_size);
Problem normalize(int rank, const int64_t* dims, const int* perm, int esize, bool fuse);
// Strided form: in_str per input dim, out_str per OUTPUT dim (elements).
Problem normalize_strided(int rank, const int64_t* dims, const int* perm, int esize,
                          const int64_t* in_str, const int64_t* out_str, bool fuse);
int widen_factor(const Problem& pr);
Problem widen_problem(const Problem& pr, int k);
tt_status_t choose_plan(Plan& plan, const DeviceInfo& dev, const tt_plan_options_t* opts,
                        OccupancyFn occ);
std::string describe_json(const Plan& plan);
int estimate_occupancy(const OccQuery& q, const DeviceInfo& dev);

// Observability (api.cu): NVTX ranges around plan / execute / the sharded
// phases (visible in Nsight timelines), and one log line per planner
// decision on stderr when tt_set_log_level(1) was called.
struct NvtxRange {
    explicit NvtxRange(const char* name);
    ~NvtxRange();
};
int log_level();
void log_plan(const Plan& p, double us, bool cached);

// api.cu --------------------------------------------------------------------
// Live-handle registry: every handle the ABI hands out (plans, contractions,
// communicators) is registered; entry points accept a handle only while it is
// registered, so a destroyed handle reads as invalid instead of as freed memory.
void* publish_handle(void* h);          // registers h (if non-null), returns it
bool handle_live(const void* h);
bool retire_handle(const void* h);      // unregisters; false if h was not live
Plan* as_plan(tt_plan_t h);
tt_status_t query_device(DeviceInfo& dev);
tt_status_t create_plan(Plan** out, int rank, const int64_t* dims, const int* perm,
                        size_t elem_size, void* stream, const DeviceInfo& dev,
                        const tt_plan_options_t* opts, OccupancyFn occ);
tt_status_t create_plan_s(Plan** out, int rank, const int64_t* dims, const int* perm,
                          size_t elem_size, void* stream, const DeviceInfo& dev,
                          const tt_plan_options_t* opts, OccupancyFn occ,
                          const int64_t* in_str, const int64_t* out_str);
tt_status_t create_plan_w(Plan** out, int rank, const int64_t* dims, const int* perm,
                          size_t elem_size, void* stream, const DeviceInfo& dev,
                          const tt_plan_options_t* opts, OccupancyFn occ, bool widenForced);
void destroy_plan(Plan* p);
constexpr size_t kPipeMinBytes = size_t(64) << 20;  // pipeline tt_execute_host above this
tt_status_t execute_host_pipelined(Plan& p, const void* host_in, void* host_out, void* dev_in,
                                   void* dev_out);

// dist.cu -------------------------------------------------------------------
void destroy_shard(ShardInfo* s);
int shard_launches(const ShardInfo* s);
std::string describe_shard_json(const Plan& plan);

// kernels.cu ----------------------------------------------------------------
int cuda_occupancy(const OccQuery& q, const DeviceInfo& dev);
int launch_plan(const Plan& plan, const void* in, void* out, void* stream);  // cudaError_t
int launch_plan_scaled(const Plan& plan, const void* in, void* out, void* stream, double alpha,
                       double beta);

}  // namespace tt
