/*
 * tt.h -- C ABI of the B200-native tensor-permutation library (libtt.so),
 * the hot path of arXiv 1705.01598 (cuTT).
 *
 * Citations: "P:Lnn" = /root/reference/PAPER.md line nn (paper text, used as
 * the specification; the library shares no code with it).
 *
 * THE OPERATION (Section 2, Eq. (1) with the output stride read as
 * c(i,O); P:L62-66 for the direction of the permutation; R1-R6):
 *
 *   A rank-n tensor with extents dims[0..n-1]; dims[0] is the stride-1
 *   (fastest) dimension ("the first tensor dimension is the stride-1
 *   dimension").  Dimensions are 0-based here (the paper is 1-based).
 *   perm[j] is the INPUT dimension that becomes OUTPUT dimension j (the
 *   paper's O = {w_j}), so the output extents are dims[perm[j]].
 *   With S_in[i] = prod_{k<i} dims[k] and S_out[j] = prod_{k<j} dims[perm[k]]:
 *
 *       out[ sum_j x[perm[j]] * S_out[j] ] = in[ sum_i x[i] * S_in[i] ]
 *
 *   for every coordinate 0 <= x[i] < dims[i].  Elements are opaque 4- or
 *   8-byte words copied bit-exactly (NaN payloads, -0.0, subnormals kept).
 *   Out-of-place only.
 *
 * API SHAPE (Section 2.3): "a plan is first created, then executed,
 * and finally destroyed, similarly to ... FFTW ... and cuFFT"; plan creation
 * "takes as input the rank and dimension extents of the input tensor, as well
 * as the permutation of the output tensor".  Unlike cuTT, a plan here owns no
 * device memory (single-GPU plans): all kernel parameters travel in the
 * launch's parameter block.
 *
 * ERRORS: every function returns tt_status_t; nothing throws across the ABI.
 * Argument errors are reported synchronously.  tt_execute is stream-ordered
 * and asynchronous: a fault inside the kernel surfaces on a later call or
 * synchronisation of the stream (as TT_CUDA_ERROR from a later tt_* call).
 *
 * THREAD SAFETY: plans are immutable after creation; concurrent tt_execute
 * calls on one single-GPU plan are safe.  A sharded plan owns staging
 * buffers and must not be executed concurrently with itself.
 */
#ifndef TT_H_
#define TT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define TT_VERSION 2
#define TT_MAX_RANK 32          /* the warp-parallel decode handles h <= 32 terms */
#define TT_NCCL_UNIQUE_ID_BYTES 128

typedef struct tt_plan_s* tt_plan_t;
typedef struct tt_comm_s* tt_comm_t;
/* A cudaStream_t (CUstream) handle; NULL means the legacy default stream. */
typedef void* tt_stream_t;

typedef enum {
    TT_SUCCESS = 0,
    TT_INVALID_PLAN = 1,        /* NULL or destroyed plan handle                    */
    TT_INVALID_PARAMETER = 2,   /* bad rank/extent/perm/pointer/in==out/alignment   */
    TT_INVALID_DEVICE = 3,      /* current device differs from the plan's device    */
    TT_UNSUPPORTED = 4,         /* elem_size not 4/8, shard extent not divisible    */
    TT_CUDA_ERROR = 5,          /* a CUDA runtime call or launch failed             */
    TT_NCCL_ERROR = 6,          /* an NCCL call failed                              */
    TT_INTERNAL_ERROR = 7,      /* allocation failure or broken invariant           */
    TT_BUFFER_TOO_SMALL = 8     /* tt_plan_describe: JSON truncated                 */
} tt_status_t;

/* Kernel families.  TT_KERNEL_AUTO lets the planner choose. */
typedef enum {
    TT_KERNEL_AUTO = 0,
    TT_KERNEL_COPY = 1,     /* rank 1 after fusion (identity): memcpy-equivalent       */
    TT_KERNEL_TILE = 2,     /* generic staged tile: Tiled / Packed / PackedSplit class  */
    TT_KERNEL_ROWCOPY = 3,  /* fastest dim unchanged, long rows: TiledCopy class        */
    TT_KERNEL_TILED2D = 4   /* two large disjoint fastest dims, 128-bit both sides      */
} tt_kernel_t;

/*
 * Optional planner overrides (tests, calibration sweeps).  Zero-initialise and
 * set only what you need; 0 always means "planner's choice".
 */
typedef struct {
    int kernel;          /* tt_kernel_t; a family that cannot run the problem -> TT_UNSUPPORTED */
    int run_in;          /* target contiguous input run, elements (TILE)          */
    int run_out;         /* target contiguous output run, elements (TILE)         */
    int threads;         /* threads per CTA (multiple of 32, <= 1024)              */
    int ctas_per_sm;     /* persistent CTAs per SM (grid = num_sms * this)         */
    int no_fusion;       /* 1 = skip dimension fusion / extent-1 removal (debug)   */
    int grid_order;      /* TILED2D tile order: 1 = A-chunks fastest, 2 = B-chunks fastest;
                            TILE: 1/0 = interleaved tiles over CTAs, 2 = contiguous ranges */
    int no_widen;        /* 1 = never regroup elements of an unchanged fastest dim into wider words */
    int stages;          /* TILE: -1 = register double buffer, 3 = cp.async 3-stage ring, 0 = planner;
                            with slot_dims = 1: 3 or 4 = slot-dim map with a cp.async ring of that
                            many stages (tile_sd_async_kernel)                                   */
    int accumulate;      /* 1 = accumulate plan for tt_execute_scaled (generic tile, 32-bit indices) */
    int slots;           /* TILE: elements per thread per tile (1, 2, 4, 8 or 16)   */
    int slot_dims;       /* TILE: 1 = slot-dim thread map when it applies, -1 = never, 0 = planner */
    int sd_vmax;         /* TILE: largest slot-dim tile searched by the model, elements
                            (<= 8192 for 4-byte, 6144 for 8-byte words); 0 = planner's default */
    int vector_gather;   /* TILE: 1 = load input runs as 16-byte chunks of their aligned superset
                            (tile_vg_kernel; stages 3/4, default 4), -1 = never, 0 = planner */
    int t2d_vec2;        /* TILED2D: 2-element vectors where the extents allow only those:
                            1 = always, -1 = never (scalar kernel), 0 = planner's measured rule */
    int force_redistribute; /* sharded plans (tt_plan_sharded_ex / _p2p_ex): take the
                            redistribution path even with one rank (single-GPU tests) */
    int vg_policy;       /* vector-gather loads, calibration: 0 = cp.async.ca (default),
                            1 = cp.async.cg (L2 only) */
    int tma;             /* TILED2D: 1 = stage the tiles with the Tensor Memory Accelerator
                            (tiled2d_tma_kernel) when every stride is a multiple of 16 bytes
                            and there are at most 3 batch dims; else TT_UNSUPPORTED */
    int a2a_chunks;      /* sharded redistribution (tt_plan_sharded_ex): cut the exchange into
                            this many chunks along the split dim so that pack, all-to-all and
                            unpack of successive chunks overlap; 1 = one serial exchange,
                            0 = planner (4 chunks from 32 MB of shard, else 1) */
} tt_plan_options_t;

/* Device description for tt_plan_offline (planning without a GPU). */
typedef struct {
    int num_sms;                 /* 148 on B200                        */
    int max_smem_per_block;      /* opt-in maximum, bytes (232448)     */
    int max_smem_per_sm;         /* bytes (233472)                     */
    int max_threads_per_sm;      /* 2048                               */
    int regs_per_sm;             /* 65536                              */
} tt_device_props_t;

/*
 * tt_plan -- create a plan for permuting a tensor of `rank` dims on the
 * CURRENT CUDA device, to be enqueued on `stream`.
 *   plan       out: receives the handle (set to NULL on failure).
 *   rank       1..TT_MAX_RANK.
 *   dims       host array [rank], every extent >= 1, product*elem_size < 2^62.
 *   perm       host array [rank], a bijection on 0..rank-1 (gather form above).
 *   elem_size  4 or 8 (else TT_UNSUPPORTED).
 *   stream     stream used by tt_execute.
 * The arrays are copied; the caller keeps ownership.  Host-only work plus
 * device-attribute queries: no device allocation, no host<->device copy.
 */
tt_status_t tt_plan(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                    size_t elem_size, tt_stream_t stream);

/*
 * tt_plan_strided -- the same permutation between caller-given layouts
 * (extension beyond P:L167, used by the fused multi-GPU redistribution):
 *     out[ sum_j x[perm[j]] * out_strides[j] ] = in[ sum_i x[i] * in_strides[i] ]
 * for every coordinate x, 0 <= x[i] < dims[i].
 *   in_strides   host array [rank], stride of INPUT dim i in elements (>= 1),
 *                or NULL for the dense column-major layout of dims.
 *   out_strides  host array [rank], stride of OUTPUT dim j in elements (>= 1),
 *                or NULL for the dense layout of the output extents.
 * The caller guarantees the output positions are distinct (no aliasing); the
 * library checks strides >= 1 and that both spans fit in 2^62 bytes.  Uses
 * the generic tile or 2-D kernels (copy, row copy and element widening need
 * dense layouts); tt_execute_host rejects non-dense plans (TT_UNSUPPORTED).
 * Executed with tt_execute (in/out = the base addresses of the two layouts).
 */
tt_status_t tt_plan_strided(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, const int64_t* in_strides,
                            const int64_t* out_strides, tt_stream_t stream);

/* tt_plan_strided without a GPU (props/opts as tt_plan_offline); describe only. */
tt_status_t tt_plan_strided_offline(tt_plan_t* plan, int rank, const int64_t* dims,
                                    const int* perm, size_t elem_size,
                                    const int64_t* in_strides, const int64_t* out_strides,
                                    const tt_device_props_t* props,
                                    const tt_plan_options_t* opts);

/* tt_plan with planner overrides (opts may be NULL = tt_plan). */
tt_status_t tt_plan_ex(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                       size_t elem_size, tt_stream_t stream, const tt_plan_options_t* opts);

/*
 * tt_plan_measure -- measurement-based plan selection ("measure the
 * runtime of tensor transpose execution for each plan and pick the fastest
 * one").  Builds the heuristic plan and up to max_candidates-1 alternatives
 * (kernel family, tile geometry, grid size; 0 = all), runs each on the device
 * buffers in/out (out is overwritten; in is only read) on `stream`, times
 * them with CUDA events and keeps the fastest.  Synchronises `stream`.
 * tt_plan_describe reports "measured": {candidates, best_ms, heuristic_ms}.
 */
tt_status_t tt_plan_measure(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, tt_stream_t stream, const void* in, void* out,
                            int max_candidates);

/*
 * tt_plan_offline -- plan for a DESCRIBED device without touching the CUDA
 * runtime (works on a machine with no GPU).  The plan can be described but
 * tt_execute on it returns TT_INVALID_DEVICE.  props may be NULL (B200 values).
 */
tt_status_t tt_plan_offline(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, const tt_device_props_t* props,
                            const tt_plan_options_t* opts);

/*
 * tt_execute -- enqueue out = permute(in) on the plan's stream.
 *   in, out  DEVICE pointers (or managed/mapped memory) of vol*elem_size
 *            bytes each, aligned to elem_size, on the plan's device.
 *            in == out -> TT_INVALID_PARAMETER (no in-place mode); other
 *            overlaps are undefined.
 * Asynchronous; does not synchronise.  Launches exactly one kernel.
 */
tt_status_t tt_execute(tt_plan_t plan, const void* in, void* out);

/*
 * tt_execute_host -- end-to-end form: copy host_in (vol*elem_size bytes,
 * preferably pinned) to the device buffer dev_in, permute into dev_out, copy
 * dev_out back to host_out, ordered after prior work on the plan's stream
 * and before later work on it.  Does not synchronise; the caller synchronises
 * the stream before reading host_out.  Above 64 MB the transfer is pipelined:
 * the output is cut into chunks along its outermost dimension, each chunk's
 * input slab is one strided 2-D H2D copy, and chunk H2D / permute / D2H run on
 * three streams so both PCIe directions and the kernels overlap (dev_in is
 * used as chunk staging).  A plan's pipeline (two streams, events, chunk
 * plans) is built on first use and freed by tt_destroy; tt_execute_host must
 * not run concurrently with itself on one plan.
 */
tt_status_t tt_execute_host(tt_plan_t plan, const void* host_in, void* host_out,
                            void* dev_in, void* dev_out);

/*
 * tt_execute_scaled -- accumulate form (SURVEY f-3, the TTC
 * comparison "read input, read output, accumulate, write output"):
 *     out = alpha * permute(in) + beta * out
 * elementwise in the element's float type (4 bytes: float, 8: double), with
 * alpha and beta converted to it, round-to-nearest multiplies and add, no
 * fused multiply-add; beta == 0 does not read out.  The plan must have been
 * created with tt_plan_options_t.accumulate = 1 (else TT_INVALID_PLAN).
 * Bandwidth convention for this form: 3 * vol * E / time.
 */
tt_status_t tt_execute_scaled(tt_plan_t plan, const void* in, void* out, double alpha, double beta);

/* tt_destroy -- free the plan (and a sharded plan's staging buffers).
 * tt_destroy(NULL) returns TT_INVALID_PLAN. */
tt_status_t tt_destroy(tt_plan_t plan);

/*
 * tt_plan_describe -- NUL-terminated JSON description of the plan written to
 * buf[len]: fused problem, kernel family, tile geometry (dims, extents,
 * strides, smem layout), grid dims, launch shape, model prediction.
 * TT_BUFFER_TOO_SMALL if it does not fit (buf then holds a truncated prefix).
 */
tt_status_t tt_plan_describe(tt_plan_t plan, char* buf, size_t len);

/* Number of kernel launches one tt_execute / tt_execute_sharded performs. */
int tt_plan_launches(tt_plan_t plan);

/* Static string for a status code. */
const char* tt_status_string(tt_status_t s);

/* TT_VERSION of the loaded library. */
int tt_version(void);

/* Planner log: level >= 1 prints one line per plan created (fused problem,
 * kernel family and variant, launch shape, model prediction, planning time,
 * plan-cache hits) to stderr; 0 (default) is silent.  Returns the previous
 * level.  (The Python binding sets it from the TT_LOG environment variable.)
 * The library also marks tt_plan / tt_execute / the sharded phases as NVTX
 * ranges for timeline tools. */
int tt_set_log_level(int level);

/* ------------------------------------------------------------------------
 * Multi-GPU (one box, one process per GPU).  The paper has no multi-GPU
 * transpose ("we will only consider local tensor transposes"); this is
 * the BASELINE.json north_star extension.
 *
 * Sharded layout: the global tensor (global_dims) is block-sharded along its
 * OUTERMOST input dimension n-1; rank r holds slab r of extent
 * global_dims[n-1]/nranks.  The output is block-sharded along its outermost
 * OUTPUT dimension n-1 (input dimension perm[n-1]) the same way.
 *   perm[n-1] == n-1 : local case, each rank permutes its slab (no traffic).
 *   otherwise        : pack (local permute) -> ncclAlltoAll over NVLink ->
 *                      unpack (local permute).
 * ---------------------------------------------------------------------- */

/* Fill id[TT_NCCL_UNIQUE_ID_BYTES] with a fresh ncclUniqueId (call on one
 * rank, broadcast the bytes, e.g. with torch.distributed). */
tt_status_t tt_comm_unique_id(void* id);

/* Create an NCCL communicator on the current device. */
tt_status_t tt_comm_init(tt_comm_t* comm, const void* nccl_unique_id, int nranks, int rank);

tt_status_t tt_comm_destroy(tt_comm_t comm);

/*
 * tt_plan_sharded -- plan the sharded permutation of a tensor of `rank` dims
 * with global extents global_dims[rank] by perm[rank] (same conventions as
 * tt_plan) on the communicator's device; the process rank and the rank count
 * come from `comm`.  global_dims[rank-1] and, for the redistribution case,
 * global_dims[perm[rank-1]] must be divisible by the number of ranks (else
 * TT_UNSUPPORTED).  The redistribution case allocates 2 x shard bytes of
 * device staging (freed by tt_destroy).
 */
tt_status_t tt_plan_sharded(tt_plan_t* plan, tt_comm_t comm, int rank, const int64_t* global_dims,
                            const int* perm, size_t elem_size, tt_stream_t stream);

/* tt_plan_sharded with options (NULL = tt_plan_sharded); only
 * force_redistribute and a2a_chunks are read. */
tt_status_t tt_plan_sharded_ex(tt_plan_t* plan, tt_comm_t comm, int rank, const int64_t* global_dims,
                               const int* perm, size_t elem_size, tt_stream_t stream,
                               const tt_plan_options_t* opts);

/*
 * tt_plan_sharded_offline -- the same geometry and sub-plans for process
 * `proc` of `nranks` without a communicator or GPU (describe only; executing
 * returns TT_INVALID_DEVICE).
 */
tt_status_t tt_plan_sharded_offline(tt_plan_t* plan, int nranks, int proc, int rank,
                                    const int64_t* global_dims, const int* perm, size_t elem_size);
/* tt_plan_sharded_offline with options (force_redistribute, a2a_chunks; NULL = defaults). */
tt_status_t tt_plan_sharded_offline_ex(tt_plan_t* plan, int nranks, int proc, int rank,
                                       const int64_t* global_dims, const int* perm, size_t elem_size,
                                       const tt_plan_options_t* opts);

/*
 * tt_execute_sharded -- local input slab -> local output slab (device
 * pointers, shard bytes each), enqueued on the plan's stream.  Collective:
 * every rank of the communicator must call it.  Local case: 1 kernel;
 * redistribution: pack kernel, ncclAlltoAll, unpack kernel -- per chunk when
 * the exchange is chunked (a2a_chunks): chunk k's pack runs on the plan's
 * stream, its all-to-all on an internal high-priority stream once that pack
 * is done, its unpack on a second internal stream once that all-to-all is
 * done, so the three steps of successive chunks overlap; the plan's stream
 * waits for the last unpack.
 */
tt_status_t tt_execute_sharded(tt_plan_t plan, const void* in_local, void* out_local);

/* Milliseconds of the last tt_execute_sharded's pack / all-to-all / unpack
 * (synchronises on that execution); zeros for the local case.  Chunked
 * exchanges report each step's span (first chunk's start to last chunk's
 * end), which overlap. */
tt_status_t tt_sharded_timings(tt_plan_t plan, float* ms3);

/* ------------------------------------------------------------------------
 * Fused redistribution (SURVEY f-1): the permutation kernels store straight
 * into the peers' output slabs over NVLink / NVSwitch -- no pack, no NCCL
 * copy, no unpack (2 x shard bytes of HBM traffic instead of ~6x).
 *
 * Geometry (same sharded layout as above; t = perm[n-1] != n-1, c =
 * global_dims[t]/nranks, j* the output position of input dim n-1): rank r's
 * slab is cut along input dim t into nranks sub-boxes x_t in [q*c, (q+1)*c);
 * sub-box q is a contiguous range of output dim j* of output slab q, at
 * y_{j*} = r*global_dims[n-1]/nranks + x_{n-1}.  Every sub-box is the same
 * strided permutation (tt_plan_strided) with different base pointers, so one
 * execute = nranks launches of one plan, own slab last.  t == n-1 is the
 * local case (one launch into the own slab).
 * ---------------------------------------------------------------------- */

/*
 * tt_plan_sharded_p2p -- fused plan for process `proc` of `nranks` (1..64)
 * on the current device.
 *   comm  NULL: single-process form -- execute with tt_execute_sharded_p2p,
 *         giving every rank's output slab as a pointer valid in this process
 *         (one process driving several GPUs with peer access enabled, or
 *         several slabs on one GPU).  Non-NULL: the multi-process form; nranks
 *         and proc must equal the communicator's (else TT_INVALID_PARAMETER);
 *         call tt_sharded_register_output once, then tt_execute_sharded.
 * Divisibility rules and errors as tt_plan_sharded.  No device allocation.
 */
tt_status_t tt_plan_sharded_p2p(tt_plan_t* plan, tt_comm_t comm, int nranks, int proc, int rank,
                                const int64_t* global_dims, const int* perm, size_t elem_size,
                                tt_stream_t stream);

/* tt_plan_sharded_p2p with options (NULL = tt_plan_sharded_p2p); only
 * force_redistribute is read (the fused path with one rank: registration and
 * both barriers run on a single GPU). */
tt_status_t tt_plan_sharded_p2p_ex(tt_plan_t* plan, tt_comm_t comm, int nranks, int proc, int rank,
                                   const int64_t* global_dims, const int* perm, size_t elem_size,
                                   tt_stream_t stream, const tt_plan_options_t* opts);

/* tt_plan_sharded_p2p geometry without a GPU (describe only): "mode" "p2p",
 * "fused" (the strided sub-box plan), "in_step" / "out_offset" (elements),
 * "dest_order". */
tt_status_t tt_plan_sharded_p2p_offline(tt_plan_t* plan, int nranks, int proc, int rank,
                                        const int64_t* global_dims, const int* perm,
                                        size_t elem_size);

/*
 * tt_sharded_register_output -- collective over the plan's communicator:
 * every rank passes the device buffer that will receive its output slab
 * (shard bytes, anywhere inside a cudaMalloc'd allocation).  CUDA IPC handles
 * of the buffers and of a small signal array (allocated here, freed by
 * tt_destroy) are all-gathered with NCCL and opened.  Once per plan; the
 * buffer must stay allocated while the plan lives.  Synchronises the plan's
 * stream.  TT_INVALID_PLAN for plans without a communicator.
 */
tt_status_t tt_sharded_register_output(tt_plan_t plan, void* out_local);

/*
 * The same registration without the communicator, for callers that exchange
 * the records themselves (and for several processes sharing one GPU, where
 * NCCL cannot form a communicator):
 *   tt_sharded_export_record -- allocate this rank's signal words and write
 *     its record (IPC handles of the allocations holding out_local and the
 *     signal words; TT_SHARD_RECORD_BYTES bytes) to the HOST buffer `record`.
 *     On failure the record is still written, flagged invalid, so peers that
 *     receive it fail too instead of waiting.
 *   tt_sharded_import_records -- `records` = the nranks records in rank
 *     order (host memory); opens every peer's handles.  Afterwards
 *     tt_execute_sharded(plan, in_local, out_local) runs the barriers and the
 *     fused stores as with a communicator.  TT_INVALID_PARAMETER if a record
 *     is flagged invalid or out of order.
 * Works on tt_plan_sharded_p2p(_ex) plans with or without a communicator.
 */
#define TT_SHARD_RECORD_BYTES 256
tt_status_t tt_sharded_export_record(tt_plan_t plan, void* out_local, void* record);
tt_status_t tt_sharded_import_records(tt_plan_t plan, const void* records);

/*
 * tt_execute_sharded_p2p -- single-process form: in_local = this process's
 * input slab (device pointer), out_slabs = host array [nranks] of every
 * rank's output slab, each writable from the plan's device.  Enqueues the
 * nranks sub-box launches on the plan's stream; NO barrier -- the caller
 * orders the ranks' executes against readers of the slabs.
 *
 * tt_execute_sharded on a registered p2p plan (out_local must be the
 * registered buffer, else TT_INVALID_PARAMETER) runs: entry barrier (every
 * peer reached this execute on its stream, so its slab is free), the
 * sub-box launches, exit barrier (every peer's stores into this slab have
 * landed).  The barriers are system-scope release/acquire signal words in
 * device memory; a peer missing for 30 s sets an error word and traps the
 * barrier kernel (the stream stops: later calls and synchronisations report
 * TT_CUDA_ERROR) instead of hanging or storing into slabs still in use.
 * tt_sharded_timings then returns (entry barrier, fused permute, exit
 * barrier) milliseconds.
 */
tt_status_t tt_execute_sharded_p2p(tt_plan_t plan, const void* in_local, void* const* out_slabs);

/* Shard geometry: local input dims and local output dims (output order),
 * `rank` entries each (either pointer may be NULL). */
tt_status_t tt_plan_shard_dims(tt_plan_t plan, int64_t* local_in_dims, int64_t* local_out_dims);

/* ------------------------------------------------------------------------
 * Tensor contraction by TTGT (SURVEY f-4; Section 3.4): the
 * workload the paper uses to show the transpose overhead inside a binary
 * contraction, D = alpha * L . R + beta * D ("D = D + L . R"), as up
 * to four transposes around one library GEMM (cuBLAS).
 *
 * Labels: modes_x[i] is the integer label (>= 0, distinct within a tensor)
 * of dimension i of tensor x (dim 0 = stride-1, as tt_plan).  A label in L
 * and R but not in D is contracted (summed); every label of D occurs in
 * exactly one of L and R (labels in all three -- batch/Hadamard -- are
 * TT_UNSUPPORTED); a label in one input only and not in D is
 * TT_INVALID_PARAMETER.  D's extents come from L and R; contracted extents
 * must match.  Elements: 4 = float, 8 = double (IEEE GEMM, no TF32).
 * ---------------------------------------------------------------------- */
typedef struct tt_contract_s* tt_contract_t;

/*
 * tt_contract_plan -- plan the contraction on the current device, enqueued on
 * `stream`.  Allocates device workspace for the operands that need a
 * transpose (vol(L), vol(R) and/or vol(D) elements; freed by
 * tt_contract_destroy) and a cuBLAS handle.  rank_d may be 0 (full
 * contraction to one element).  m, n, k >= 2^31 -> TT_UNSUPPORTED.
 */
tt_status_t tt_contract_plan(tt_contract_t* plan, int rank_d, const int* modes_d, int rank_l,
                             const int64_t* dims_l, const int* modes_l, int rank_r,
                             const int64_t* dims_r, const int* modes_r, size_t elem_size,
                             tt_stream_t stream);

/* Same without a GPU (describe only; execute returns TT_INVALID_DEVICE). */
tt_status_t tt_contract_plan_offline(tt_contract_t* plan, int rank_d, const int* modes_d,
                                     int rank_l, const int64_t* dims_l, const int* modes_l,
                                     int rank_r, const int64_t* dims_r, const int* modes_r,
                                     size_t elem_size);

/*
 * tt_contract_execute -- D = alpha * L . R + beta * D (device pointers, dense
 * column-major tensors, aligned to elem_size; D distinct from L and R).
 * Stream-ordered, asynchronous.  beta != 0 with a back transpose needs the
 * accumulate form (32-bit indices) -- else TT_UNSUPPORTED.
 */
tt_status_t tt_contract_execute(tt_contract_t plan, const void* l, const void* r, void* d,
                                double alpha, double beta);

/* Milliseconds of the last execute's steps: transpose L, transpose R, GEMM,
 * transpose D (zero for skipped steps; synchronises on that execute). */
tt_status_t tt_contract_timings(tt_contract_t plan, float* ms4);

/* JSON: m, n, k, which transposes run, GEMM ops, sub-plans. */
tt_status_t tt_contract_describe(tt_contract_t plan, char* buf, size_t len);

tt_status_t tt_contract_destroy(tt_contract_t plan);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* TT_H_ */
