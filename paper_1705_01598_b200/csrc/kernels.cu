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
//
// This file: the launch layer (occupancy queries, dynamic shared-memory
// attributes, plan -> kernel dispatch).  The kernels live in kernels_*.cu.
#include <cuda_runtime.h>

#include <cstdint>
#include <cuda.h>
#include <mutex>
#include <unordered_map>
#include <unordered_set>

#include "tt_internal.h"
#include "kern_pick.h"

namespace tt {

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

struct OccKey {
    const void* fn;
    int threads, smem, device;
    bool operator==(const OccKey& o) const {
        return fn == o.fn && threads == o.threads && smem == o.smem && device == o.device;
    }
};
struct OccKeyHash {
    size_t operator()(const OccKey& k) const {
        return std::hash<const void*>()(k.fn) ^ ((size_t)k.threads << 1) ^ ((size_t)k.smem << 12) ^
               ((size_t)k.device << 40);
    }
};
static std::mutex g_occ_mu;
static std::unordered_map<OccKey, int, OccKeyHash> g_occ;

int cuda_occupancy(const OccQuery& q, const DeviceInfo& dev) {
    (void)dev;
    const void* fn = q.tma ? pick_tiled2d_tma(q.esize, q.tma)
                     : q.kernel == TT_KERNEL_TILE
                         ? (q.vg ? pick_tile_vg(q.esize, q.nreg, q.vg, q.vec, q.threads)
                            : q.sdq ? pick_tile_sd(q.esize, q.sdq, q.sdr, q.vec >= 3 ? q.vec : 0)
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
    // one CUDA query per (kernel, launch shape, device) and process: planning
    // asks the same questions many times (candidates, re-plans)
    int devn = 0;
    if (cudaGetDevice(&devn) != cudaSuccess) { cudaGetLastError(); return 0; }
    const OccKey key{fn, q.threads, q.smem, devn};
    {
        std::lock_guard<std::mutex> g(g_occ_mu);
        auto it = g_occ.find(key);
        if (it != g_occ.end()) return it->second;
    }
    if (ensure_max_smem(fn) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int blocks = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, q.threads, q.smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    std::lock_guard<std::mutex> g(g_occ_mu);
    g_occ[key] = blocks;
    return blocks;
}

// TMA tensor maps hold the global address: encoded for each (in, out) pair
// (cuTensorMapEncodeTiled through the driver entry point), the last pair
// cached in the plan.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(f);
        cudaGetLastError();
    });
    return fn;
}

static bool encode_maps(const Tma2DParams& t, int E, const void* in, void* out, CUtensorMap* mi, CUtensorMap* mo) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const CUtensorMapDataType dt = E == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_INT64;
    const cuuint32_t boxIn[5] = {(cuuint32_t)t.TA, (cuuint32_t)t.TB, 1, 1, 1};
    const cuuint32_t boxOut[5] = {(cuuint32_t)t.TB, (cuuint32_t)t.TA, 1, 1, 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (fn(mi, dt, (cuuint32_t)t.rank, const_cast<void*>(in), t.gDimIn, t.gStrideIn, boxIn, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    return fn(mo, dt, (cuuint32_t)t.rank, out, t.gDimOut, t.gStrideOut, boxOut, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int launch_tma(const Plan& plan, const void* in, void* out, cudaStream_t stream) {
    const KernelChoice& kc = plan.kc;
    const int E = plan.prob.esize;
    // TMA needs 16-byte-aligned global addresses
    if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) != 0)
        return (int)cudaErrorMisalignedAddress;
    Tma2DParams p = plan.tma;
    Plan::TmaCache* c = plan.tmaCache;
    bool ok = false;
    if (c) {
        std::lock_guard<std::mutex> g(c->mu);
        if (c->in == in && c->out == out) {
            p.inMap = c->inMap;
            p.outMap = c->outMap;
            ok = true;
        } else if (encode_maps(plan.tma, E, in, out, &p.inMap, &p.outMap)) {
            c->in = in;
            c->out = out;
            c->inMap = p.inMap;
            c->outMap = p.outMap;
            ok = true;
        }
    } else {
        ok = encode_maps(plan.tma, E, in, out, &p.inMap, &p.outMap);
    }
    if (!ok) return (int)cudaErrorInvalidValue;
    const void* fn = pick_tiled2d_tma(E, p.rank);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    cudaError_t e = ensure_max_smem(fn);
    if (e != cudaSuccess) return (int)e;
    void* args[] = {(void*)&p};
    return (int)cudaLaunchKernel(fn, dim3(kc.grid), dim3(kc.threads), args, kc.smem, stream);
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
        void* args[] = {(void*)&in, (void*)&out, (void*)&n, (void*)&vec16};
        return (int)cudaLaunchKernel(pick_copy(), dim3(kc.grid), dim3(kc.threads), args, 0, stream);
    }
    if (kc.kernel == TT_KERNEL_ROWCOPY) {
        const void* fn = pick_rowcopy(E, kc.idx64);
        if (!fn) return (int)cudaErrorInvalidConfiguration;
        void* args[] = {(void*)&plan.row, (void*)&in, (void*)&out};
        return (int)cudaLaunchKernel(fn, dim3(kc.grid), dim3(kc.threads), args, 0, stream);
    }
    if (kc.tma) return launch_tma(plan, in, out, stream);
    if (kc.kernel == TT_KERNEL_TILE || kc.kernel == TT_KERNEL_TILED2D) {
        bool t2 = kc.kernel == TT_KERNEL_TILED2D;
        int threads = kc.threads, grid = kc.grid, smem = kc.smem, stages = kc.stages;
        if (t2 && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) &
                   (uintptr_t)(kc.vec * E - 1)) != 0) {
            // pointers not aligned to the vector width: generic tile fallback
            t2 = false;
            threads = kc.fb_threads;
            grid = kc.fb_grid;
            smem = kc.fb_smem;
            stages = kc.fb_stages;
        }
        const void* fn = t2 ? (kc.vec == 1 && kc.stages >= 3 && !kc.idx64
                                   ? pick_tiled2d_async(E, kc.tile0, kc.tile1, kc.stages)
                                   : pick_tiled2d(E, kc.vec, kc.tile0, kc.tile1, kc.idx64))
                            : kc.vg ? pick_tile_vg(E, kc.nreg, plan.tile.vgK, stages, threads)
                            : kc.sdq ? pick_tile_sd(E, kc.sdq, kc.sdr, stages)
                            : kc.acc ? pick_tile_acc(E, kc.nreg)
                                     : (stages >= 3 ? pick_tile_async(E, kc.nreg, kc.idx64)
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
