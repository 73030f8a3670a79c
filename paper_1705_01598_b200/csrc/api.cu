// api.cu -- the C ABI declared in include/tt.h (plan -> execute -> destroy,
// P:L167).  Argument marshalling, device queries and launches only; the
// planner lives in planner.cpp and the kernels in kernels.cu.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <algorithm>
#include <list>
#include <unordered_map>
#include <mutex>
#include <unordered_set>

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <chrono>

#include "tt_internal.h"

using namespace tt;

namespace tt {

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

static std::atomic<int> g_log_level{0};
int log_level() { return g_log_level.load(std::memory_order_relaxed); }

void log_plan(const Plan& p, double us, bool cached) {
    const Problem& pr = p.prob;
    const KernelChoice& kc = p.kc;
    std::string f = "[";
    for (int i = 0; i < pr.n; ++i) f += (i ? "," : "") + std::to_string(pr.d[i]);
    f += "] perm [";
    for (int i = 0; i < pr.n; ++i) f += (i ? "," : "") + std::to_string(pr.p[i]);
    f += "]";
    const char* k = kc.kernel == TT_KERNEL_COPY ? "copy" : kc.kernel == TT_KERNEL_ROWCOPY ? "rowcopy"
                    : kc.kernel == TT_KERNEL_TILED2D ? "tiled2d" : "tile";
    const char* var = kc.kernel != TT_KERNEL_TILE ? "" : kc.vg ? "/vector-gather" : kc.sdq ? "/slot-dim" : "/classic";
    std::fprintf(stderr,
                 "[tt] plan rank %d E %d -> fused %s word %dB: %s%s threads %d grid %d smem %d slots %d "
                 "stages %d tile V %d predicted %.1f us, planned in %.1f us%s\n",
                 p.rank, pr.esize / p.widen, f.c_str(), pr.esize, k, var, kc.threads, kc.grid, kc.smem,
                 kc.nreg, kc.stages, kc.kernel == TT_KERNEL_TILE ? p.tile.V : 0, kc.predicted_us, us,
                 cached ? " (plan cache)" : "");
}

static std::mutex g_handles_mu;
static std::unordered_set<const void*> g_handles;

void* publish_handle(void* h) {
    if (h != nullptr) {
        std::lock_guard<std::mutex> g(g_handles_mu);
        g_handles.insert(h);
    }
    return h;
}

bool handle_live(const void* h) {
    if (h == nullptr) return false;
    std::lock_guard<std::mutex> g(g_handles_mu);
    return g_handles.count(h) != 0;
}

bool retire_handle(const void* h) {
    if (h == nullptr) return false;
    std::lock_guard<std::mutex> g(g_handles_mu);
    return g_handles.erase(h) != 0;
}

Plan* as_plan(tt_plan_t h) {
    return handle_live(h) ? reinterpret_cast<Plan*>(h) : nullptr;
}

static std::mutex g_dev_mu;
static std::unordered_map<int, DeviceInfo> g_dev;

tt_status_t query_device(DeviceInfo& dev) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    {
        std::lock_guard<std::mutex> g(g_dev_mu);
        auto it = g_dev.find(d);
        if (it != g_dev.end()) { dev = it->second; return TT_SUCCESS; }
    }
    dev.device = d;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
        cudaGetLastError();
        return TT_INVALID_DEVICE;
    }
    dev.num_sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d) == cudaSuccess)
        dev.max_smem_per_block = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, d) == cudaSuccess)
        dev.max_smem_per_sm = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxThreadsPerMultiProcessor, d) == cudaSuccess)
        dev.max_threads_per_sm = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxRegistersPerMultiprocessor, d) == cudaSuccess)
        dev.regs_per_sm = v;
    cudaGetLastError();
    std::lock_guard<std::mutex> g(g_dev_mu);
    g_dev[d] = dev;
    return TT_SUCCESS;
}

// ---------------------------------------------------------------------------
// Plan cache: planning is pure host work whose result depends only on the
// problem, the options and the device, so tt_plan of a problem seen before
// (LRU of 64) copies the earlier decision instead of searching again -- the
// one-shot transposes of P:L167 pay the search once per process.
// ---------------------------------------------------------------------------
static Plan* clone_plan(const Plan& src) {
    Plan* p = new (std::nothrow) Plan();
    if (p == nullptr) return nullptr;
    p->device = src.device;
    p->stream = src.stream;
    p->rank = src.rank;
    p->dims = src.dims;
    p->perm = src.perm;
    p->prob = src.prob;
    p->kc = src.kc;
    p->tile = src.tile;
    p->row = src.row;
    p->t2d = src.t2d;
    p->tma = src.tma;
    if (src.tmaCache) p->tmaCache = new (std::nothrow) Plan::TmaCache();
    p->widen = src.widen;
    if (src.narrow) {
        p->narrow = clone_plan(*src.narrow);
        if (p->narrow == nullptr) { delete p; return nullptr; }
    }
    return p;
}

struct PlanCache {
    std::mutex mu;
    std::list<std::pair<std::string, Plan*>> lru;  // front = most recent
    std::unordered_map<std::string, std::list<std::pair<std::string, Plan*>>::iterator> map;
    static constexpr size_t kCap = 64;
    ~PlanCache() {
        for (auto& e : lru) destroy_plan(e.second);
    }
};
static PlanCache g_cache;

static std::string cache_key(int rank, const int64_t* dims, const int* perm, size_t elem_size,
                             const DeviceInfo& dev, const tt_plan_options_t* opts) {
    std::string k;
    k.append(reinterpret_cast<const char*>(&dev), sizeof(dev));
    k.append(reinterpret_cast<const char*>(&rank), sizeof(rank));
    k.append(reinterpret_cast<const char*>(&elem_size), sizeof(elem_size));
    k.append(reinterpret_cast<const char*>(dims), sizeof(int64_t) * rank);
    k.append(reinterpret_cast<const char*>(perm), sizeof(int) * rank);
    tt_plan_options_t o{};
    if (opts) o = *opts;
    k.append(reinterpret_cast<const char*>(&o), sizeof(o));
    return k;
}

static Plan* cache_get(const std::string& key, void* stream) {
    std::lock_guard<std::mutex> g(g_cache.mu);
    auto it = g_cache.map.find(key);
    if (it == g_cache.map.end()) return nullptr;
    g_cache.lru.splice(g_cache.lru.begin(), g_cache.lru, it->second);
    Plan* p = clone_plan(*it->second->second);
    if (p) {
        p->stream = stream;
        if (p->narrow) p->narrow->stream = stream;
    }
    return p;
}

static void cache_put(const std::string& key, const Plan& plan) {
    Plan* c = clone_plan(plan);
    if (c == nullptr) return;
    std::lock_guard<std::mutex> g(g_cache.mu);
    if (g_cache.map.count(key)) { destroy_plan(c); return; }
    g_cache.lru.emplace_front(key, c);
    g_cache.map[key] = g_cache.lru.begin();
    if (g_cache.lru.size() > PlanCache::kCap) {
        auto& last = g_cache.lru.back();
        g_cache.map.erase(last.first);
        destroy_plan(last.second);
        g_cache.lru.pop_back();
    }
}

tt_status_t create_plan(Plan** out, int rank, const int64_t* dims, const int* perm,
                        size_t elem_size, void* stream, const DeviceInfo& dev,
                        const tt_plan_options_t* opts, OccupancyFn occ) {
    return create_plan_w(out, rank, dims, perm, elem_size, stream, dev, opts, occ, false);
}

tt_status_t create_plan_s(Plan** out, int rank, const int64_t* dims, const int* perm,
                          size_t elem_size, void* stream, const DeviceInfo& dev,
                          const tt_plan_options_t* opts, OccupancyFn occ,
                          const int64_t* in_str, const int64_t* out_str) {
    if (in_str == nullptr && out_str == nullptr)
        return create_plan_w(out, rank, dims, perm, elem_size, stream, dev, opts, occ, false);
    if (out == nullptr) return TT_INVALID_PARAMETER;
    *out = nullptr;
    tt_status_t st = validate(rank, dims, perm, elem_size);
    if (st != TT_SUCCESS) return st;
    if (opts && (opts->accumulate || opts->stages >= 3)) return TT_UNSUPPORTED;
    // dense defaults for the side not given; strides >= 1 (no broadcast: the
    // map must stay one-to-one on the output)
    int64_t si[kMaxDims], so[kMaxDims];
    int64_t acc = 1;
    for (int i = 0; i < rank; ++i) { si[i] = in_str ? in_str[i] : acc; acc *= dims[i]; }
    acc = 1;
    for (int j = 0; j < rank; ++j) { so[j] = out_str ? out_str[j] : acc; acc *= dims[perm[j]]; }
    long double maxIn = 0, maxOut = 0;
    for (int i = 0; i < rank; ++i) {
        if (si[i] < 1 || so[i] < 1) return TT_INVALID_PARAMETER;
        maxIn += (long double)(dims[i] - 1) * si[i];
        maxOut += (long double)(dims[perm[i]] - 1) * so[i];
    }
    if ((maxIn + 1) * elem_size >= (long double)(1LL << 62) ||
        (maxOut + 1) * elem_size >= (long double)(1LL << 62))
        return TT_INVALID_PARAMETER;
    Plan* p = new (std::nothrow) Plan();
    if (p == nullptr) return TT_INTERNAL_ERROR;
    p->device = dev.device;
    p->stream = stream;
    p->rank = rank;
    p->dims.assign(dims, dims + rank);
    p->perm.assign(perm, perm + rank);
    p->prob = normalize_strided(rank, dims, perm, (int)elem_size, si, so, !(opts && opts->no_fusion));
    st = choose_plan(*p, dev, opts, occ);
    if (st != TT_SUCCESS) {
        delete p;
        return st;
    }
    if (p->kc.tma) p->tmaCache = new (std::nothrow) Plan::TmaCache();
    *out = p;
    return TT_SUCCESS;
}

tt_status_t create_plan_w(Plan** out, int rank, const int64_t* dims, const int* perm,
                          size_t elem_size, void* stream, const DeviceInfo& dev,
                          const tt_plan_options_t* opts, OccupancyFn occ, bool widenForced) {
    if (out == nullptr) return TT_INVALID_PARAMETER;
    *out = nullptr;
    tt_status_t st = validate(rank, dims, perm, elem_size);
    if (st != TT_SUCCESS) return st;
    if (opts && opts->slots != 0 && opts->slots != 1 && opts->slots != 2 && opts->slots != 4 &&
        opts->slots != 8 && opts->slots != 16)
        return TT_INVALID_PARAMETER;
    Plan* p = new (std::nothrow) Plan();
    if (p == nullptr) return TT_INTERNAL_ERROR;
    p->device = dev.device;
    p->stream = stream;
    p->rank = rank;
    p->dims.assign(dims, dims + rank);
    p->perm.assign(perm, perm + rank);
    const bool fuse = !(opts && opts->no_fusion);
    p->prob = normalize(rank, dims, perm, (int)elem_size, fuse);
    // element widening (planner.cpp widen_factor) unless geometry is forced
    const bool forcedGeometry = opts && (opts->no_widen || opts->accumulate ||
                                         (!widenForced && (opts->kernel || opts->run_in ||
                                                           opts->run_out || opts->threads || opts->slots)));
    const int k = forcedGeometry ? 1 : widen_factor(p->prob);
    if (k > 1) {
        Plan* nar = new (std::nothrow) Plan();
        if (nar == nullptr) { delete p; return TT_INTERNAL_ERROR; }
        nar->device = p->device;
        nar->stream = p->stream;
        nar->rank = rank;
        nar->dims = p->dims;
        nar->perm = p->perm;
        nar->prob = p->prob;
        if (choose_plan(*nar, dev, opts, occ) == TT_SUCCESS) {
            p->narrow = nar;
            p->widen = k;
            p->prob = widen_problem(p->prob, k);
        } else {
            delete nar;
        }
    }
    st = choose_plan(*p, dev, opts, occ);
    if (st != TT_SUCCESS) {
        delete p;
        return st;
    }
    // 8-byte elements whose rows the row copy would move as widened 16-byte
    // words: the un-widened generic tile is faster (same-box A/B over the
    // suites' row-copy cases, profiles/round2_ab_rowcopy_tile/: 9 of 9 such
    // cases 0.89-0.94x the time; un-widened 8-byte rows were mixed and keep
    // the row copy; so do problems of fewer than 8192 rows -- e.g. the
    // sharded unpack's few long rows -- which the A/B did not cover).
    // Planner-chosen plans only.
    static const tt_plan_options_t zeroOpts{};
    const bool noOpts = opts == nullptr || std::memcmp(opts, &zeroOpts, sizeof(zeroOpts)) == 0;
    if (noOpts && elem_size == 8 && p->widen > 1 && p->kc.kernel == TT_KERNEL_ROWCOPY &&
        p->row.nRows / std::max<int64_t>(1, p->row.nseg) >= 8192) {
        Plan* t = new (std::nothrow) Plan();
        if (t != nullptr) {
            t->device = p->device;
            t->stream = p->stream;
            t->rank = rank;
            t->dims = p->dims;
            t->perm = p->perm;
            t->prob = normalize(rank, dims, perm, (int)elem_size, !(opts && opts->no_fusion));
            tt_plan_options_t o{};
            o.kernel = TT_KERNEL_TILE;
            if (choose_plan(*t, dev, &o, occ) == TT_SUCCESS) {
                delete p;
                p = t;
            } else {
                delete t;
            }
        }
    }
    if (p->kc.tma) p->tmaCache = new (std::nothrow) Plan::TmaCache();
    *out = p;
    return TT_SUCCESS;
}

// ---------------------------------------------------------------------------
// Pipelined host path of tt_execute_host: the output is cut into chunks
// along its OUTERMOST dim (input dim t = perm[n-1]); output chunk q is a
// contiguous block, and its input is the slab x_t in chunk q -- a strided 2-D
// region of the host input (width c*S_in[t], pitch d_t*S_in[t]).  Chunk q's
// H2D (one cudaMemcpy2DAsync), its permutation (a plan of the chunk problem)
// and its D2H run on three streams linked by events, so the two PCIe
// directions and the kernels overlap.
// ---------------------------------------------------------------------------
struct HostPipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev;   // 3 per chunk: in-ready, out-ready, +1 start/end
    int nchunks = 0;
    int64_t chunk = 0, tail = 0;
    Plan* full = nullptr;
    Plan* last = nullptr;
    int device = -1;
    ~HostPipe() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        destroy_plan(full);
        if (last != full) destroy_plan(last);
    }
};

static tt_status_t build_pipe(Plan& p) {
    const int n = p.rank;
    const int t = p.perm[n - 1];
    const int64_t dt = p.dims[t];
    if (dt < 2) return TT_UNSUPPORTED;
    // chunks of >= 16 MB, at most 32 (S1 e2e: 4 / 8 / 16 / 32 chunks =
    // 82 / 88 / 90 / 92 GB/s -- both PCIe directions near their limit; more
    // chunks shorten the pipeline's fill and drain)
    int64_t volAll = 1;
    for (int64_t x : p.dims) volAll *= x;
    const int64_t bytesAll = volAll * (p.prob.esize / p.widen);
    const int want = (int)std::max<int64_t>(2, std::min<int64_t>(32, bytesAll >> 24));
    const int nch = (int)std::min<int64_t>(dt, want);
    HostPipe* hp = new (std::nothrow) HostPipe();
    if (!hp) return TT_INTERNAL_ERROR;
    hp->device = p.device;
    hp->chunk = (dt + nch - 1) / nch;
    hp->nchunks = (int)((dt + hp->chunk - 1) / hp->chunk);
    hp->tail = dt - (int64_t)(hp->nchunks - 1) * hp->chunk;
    DeviceInfo dev;
    if (query_device(dev) != TT_SUCCESS) { delete hp; return TT_CUDA_ERROR; }
    const int esize = p.prob.esize / p.widen;
    std::vector<int64_t> cd(p.dims);
    cd[t] = hp->chunk;
    if (create_plan(&hp->full, n, cd.data(), p.perm.data(), esize, p.stream, dev, nullptr,
                    &cuda_occupancy) != TT_SUCCESS) { delete hp; return TT_UNSUPPORTED; }
    if (hp->tail != hp->chunk) {
        cd[t] = hp->tail;
        if (create_plan(&hp->last, n, cd.data(), p.perm.data(), esize, p.stream, dev, nullptr,
                        &cuda_occupancy) != TT_SUCCESS) { delete hp; return TT_UNSUPPORTED; }
    } else {
        hp->last = hp->full;
    }
    if (cudaStreamCreateWithFlags(&hp->h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hp->d2h, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        delete hp;
        return TT_CUDA_ERROR;
    }
    hp->ev.assign(2 * hp->nchunks + 2, nullptr);
    for (auto& e : hp->ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            delete hp;
            return TT_CUDA_ERROR;
        }
    p.pipe = hp;
    return TT_SUCCESS;
}

tt_status_t execute_host_pipelined(Plan& p, const void* host_in, void* host_out, void* dev_in,
                                   void* dev_out) {
    if (p.pipe == nullptr) {
        tt_status_t st = build_pipe(p);
        if (st != TT_SUCCESS) return st;
    }
    HostPipe* hp = p.pipe;
    const int n = p.rank;
    const int t = p.perm[n - 1];
    const size_t E = (size_t)(p.prob.esize / p.widen);
    int64_t sIn = 1;  // input stride of dim t
    for (int i = 0; i < t; ++i) sIn *= p.dims[i];
    int64_t vol = 1;
    for (int i = 0; i < n; ++i) vol *= p.dims[i];
    const int64_t dt = p.dims[t];
    const int64_t rows = vol / (dt * sIn);  // product of the dims after t
    const int64_t outBlock = vol / dt;      // output elements per unit of x_t
    cudaStream_t main = static_cast<cudaStream_t>(p.stream);
    cudaEvent_t start = hp->ev[2 * hp->nchunks], done = hp->ev[2 * hp->nchunks + 1];
    bool ok = cudaEventRecord(start, main) == cudaSuccess &&
              cudaStreamWaitEvent(hp->h2d, start, 0) == cudaSuccess &&
              cudaStreamWaitEvent(hp->d2h, start, 0) == cudaSuccess;
    for (int q = 0; ok && q < hp->nchunks; ++q) {
        const int64_t c = (q == hp->nchunks - 1) ? hp->tail : hp->chunk;
        const int64_t x0 = (int64_t)q * hp->chunk;
        char* dIn = static_cast<char*>(dev_in) + (size_t)(x0 * sIn * rows) * E;
        const char* hIn = static_cast<const char*>(host_in) + (size_t)(x0 * sIn) * E;
        ok = cudaMemcpy2DAsync(dIn, (size_t)(c * sIn) * E, hIn, (size_t)(dt * sIn) * E,
                               (size_t)(c * sIn) * E, (size_t)rows, cudaMemcpyHostToDevice,
                               hp->h2d) == cudaSuccess &&
             cudaEventRecord(hp->ev[2 * q], hp->h2d) == cudaSuccess &&
             cudaStreamWaitEvent(main, hp->ev[2 * q], 0) == cudaSuccess;
        if (!ok) break;
        char* dOut = static_cast<char*>(dev_out) + (size_t)(x0 * outBlock) * E;
        Plan* cp = (q == hp->nchunks - 1) ? hp->last : hp->full;
        ok = launch_plan(*cp, dIn, dOut, p.stream) == 0 &&
             cudaEventRecord(hp->ev[2 * q + 1], main) == cudaSuccess &&
             cudaStreamWaitEvent(hp->d2h, hp->ev[2 * q + 1], 0) == cudaSuccess &&
             cudaMemcpyAsync(static_cast<char*>(host_out) + (size_t)(x0 * outBlock) * E, dOut,
                             (size_t)(c * outBlock) * E, cudaMemcpyDeviceToHost, hp->d2h) == cudaSuccess;
    }
    ok = ok && cudaEventRecord(done, hp->d2h) == cudaSuccess &&
         cudaStreamWaitEvent(main, done, 0) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    return TT_SUCCESS;
}

Plan::~Plan() {
    delete tmaCache;
    delete narrow;
    delete pipe;
}

void destroy_plan(Plan* p) {
    if (p == nullptr) return;
    if (p->shard) destroy_shard(p->shard);
    p->shard = nullptr;
    delete p;
}

}  // namespace tt

static tt_status_t make_plan(tt_plan_t* out, int rank, const int64_t* dims, const int* perm,
                             size_t elem_size, tt_stream_t stream, const DeviceInfo& dev,
                             const tt_plan_options_t* opts, OccupancyFn occ) {
    NvtxRange nv("tt_plan");
    const auto t0 = std::chrono::steady_clock::now();
    auto us = [&]() {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    };
    Plan* p = nullptr;
    const bool cacheable = dev.device >= 0;  // device plans (validated below before insertion)
    std::string key;
    if (cacheable) {
        key = cache_key(rank, dims, perm, elem_size, dev, opts);
        p = cache_get(key, stream);
        if (p != nullptr) {
            if (log_level() > 0) log_plan(*p, us(), true);
            if (out) *out = reinterpret_cast<tt_plan_t>(publish_handle(p));
            return TT_SUCCESS;
        }
    }
    tt_status_t st = create_plan(&p, rank, dims, perm, elem_size, stream, dev, opts, occ);
    if (st == TT_SUCCESS) p->plan_us = us();
    if (st == TT_SUCCESS && log_level() > 0) log_plan(*p, us(), false);
    if (st == TT_SUCCESS && cacheable) cache_put(key, *p);
    if (out) *out = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return st;
}

static tt_status_t check_exec(Plan* p, const void* in, void* out) {
    if (p == nullptr) return TT_INVALID_PLAN;
    if (in == nullptr || out == nullptr || in == out) return TT_INVALID_PARAMETER;
    const uintptr_t mis = (reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) &
                          (uintptr_t)(p->prob.esize / p->widen - 1);
    if (mis) return TT_INVALID_PARAMETER;
    if (p->device < 0) return TT_INVALID_DEVICE;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    if (d != p->device) return TT_INVALID_DEVICE;
    return TT_SUCCESS;
}


extern "C" {

int tt_version(void) { return TT_VERSION; }

int tt_set_log_level(int level) {
    return g_log_level.exchange(level < 0 ? 0 : level);
}

const char* tt_status_string(tt_status_t s) {
    switch (s) {
        case TT_SUCCESS: return "TT_SUCCESS";
        case TT_INVALID_PLAN: return "TT_INVALID_PLAN";
        case TT_INVALID_PARAMETER: return "TT_INVALID_PARAMETER";
        case TT_INVALID_DEVICE: return "TT_INVALID_DEVICE";
        case TT_UNSUPPORTED: return "TT_UNSUPPORTED";
        case TT_CUDA_ERROR: return "TT_CUDA_ERROR";
        case TT_NCCL_ERROR: return "TT_NCCL_ERROR";
        case TT_INTERNAL_ERROR: return "TT_INTERNAL_ERROR";
        case TT_BUFFER_TOO_SMALL: return "TT_BUFFER_TOO_SMALL";
        default: return "TT_UNKNOWN_STATUS";
    }
}

tt_status_t tt_plan_ex(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                       size_t elem_size, tt_stream_t stream, const tt_plan_options_t* opts) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    tt_status_t st = validate(rank, dims, perm, elem_size);
    if (st != TT_SUCCESS) return st;
    DeviceInfo dev;
    st = query_device(dev);
    if (st != TT_SUCCESS) return st;
    return make_plan(plan, rank, dims, perm, elem_size, stream, dev, opts, &cuda_occupancy);
}

tt_status_t tt_plan(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                    size_t elem_size, tt_stream_t stream) {
    return tt_plan_ex(plan, rank, dims, perm, elem_size, stream, nullptr);
}

// Measurement-based plan selection ("measure the runtime of tensor
// transpose execution for each plan and pick the fastest one"): the
// heuristic plan plus alternative kernels / tile geometries / grid sizes are
// each run on (in, out) and timed with CUDA events on the plan's stream.
tt_status_t tt_plan_measure(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, tt_stream_t stream, const void* in, void* out,
                            int max_candidates) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    tt_status_t st = validate(rank, dims, perm, elem_size);
    if (st != TT_SUCCESS) return st;
    if (in == nullptr || out == nullptr || in == out) return TT_INVALID_PARAMETER;
    DeviceInfo dev;
    st = query_device(dev);
    if (st != TT_SUCCESS) return st;
    Plan* heur = nullptr;
    st = create_plan(&heur, rank, dims, perm, elem_size, stream, dev, nullptr, &cuda_occupancy);
    if (st != TT_SUCCESS) return st;
    // the execute-time checks (alignment, device) before any candidate runs
    st = check_exec(heur, in, out);
    if (st != TT_SUCCESS) { destroy_plan(heur); return st; }

    // candidate options (elements of the widened problem when it widens)
    std::vector<tt_plan_options_t> vars;
    auto opt = [](int kernel, int a, int b, int threads, int cps, int order) {
        tt_plan_options_t o;
        std::memset(&o, 0, sizeof(o));
        o.kernel = kernel; o.run_in = a; o.run_out = b; o.threads = threads;
        o.ctas_per_sm = cps; o.grid_order = order;
        return o;
    };
    const Problem& hp = heur->prob;
    const int W = hp.esize;
    // 2-D candidates only when the two fastest dims fill 64 x 64 tiles
    // reasonably: forced on, say, a 2 x 2 pair the 2-D kernel is correct but
    // ~2000x slower (every tile nearly empty), which made measuring a rank-12
    // problem take 80 s
    auto fill64 = [&](int64_t d) { return (double)d / (64.0 * (double)((d + 63) / 64)); };
    const bool t2dSane = hp.n >= 2 && hp.p[0] != 0 && fill64(hp.d[0]) * fill64(hp.d[hp.p[0]]) >= 0.25;
    if (t2dSane) {
        const int tiles4[4][2] = {{64, 128}, {128, 64}, {128, 128}, {64, 64}};
        const int tiles8[4][2] = {{64, 64}, {64, 32}, {32, 64}, {32, 32}};
        for (int t = 0; t < 4; ++t)
            for (int cps : {1, 2, 3, 4})
                for (int st : {0, 4}) {  // stages 4: the scalar kernel's cp.async ring
                    tt_plan_options_t o = W == 4 ? opt(TT_KERNEL_TILED2D, tiles4[t][0], tiles4[t][1], 0, cps, 2)
                                                 : opt(TT_KERNEL_TILED2D, tiles8[t][0], tiles8[t][1], 0, cps, 2);
                    o.stages = st;
                    vars.push_back(o);
                }
    }
    if (hp.n >= 2 && hp.p[0] == 0)
        for (int cps : {2, 4, 8}) vars.push_back(opt(TT_KERNEL_ROWCOPY, 0, 0, 0, cps, 0));
    if (hp.n >= 2)
        for (int bi : {128, 256, 512, 1024})
            for (int bo : {128, 256, 512, 1024})
                vars.push_back(opt(TT_KERNEL_TILE, std::max(2, bi / W), std::max(2, bo / W), 0, 0, 0));
    // whole-dimension prefix products as run targets (tiles without split
    // dims; the heuristic takes them only when they keep the output run)
    if (hp.n >= 2 && hp.p[0] != 0) {
        std::vector<int64_t> pin, pout;
        int64_t P = 1;
        for (int i = 0; i < hp.n && P * hp.d[i] <= 4096; ++i) { P *= hp.d[i]; if (P >= 8) pin.push_back(P); }
        P = 1;
        for (int j = 0; j < hp.n && P * hp.d[hp.p[j]] <= 4096; ++j) {
            P *= hp.d[hp.p[j]];
            if (P >= 8) pout.push_back(P);
        }
        for (int64_t a : pin)
            for (int64_t b : pout) vars.push_back(opt(TT_KERNEL_TILE, (int)a, (int)b, 0, 0, 0));
    }
    // larger slot-dim tiles (up to 8192 elements; whole short dims instead of
    // split ones): won up to 1.6x on Set-2 shapes and lost elsewhere, which the
    // model cannot rank -- measurement can (tools/tile_runs_sweep.py)
    if (hp.n >= 2 && hp.p[0] != 0)
        for (int bi : {64, 128, 256, 512})
            for (int bo : {64, 128, 256, 512}) {
                tt_plan_options_t o = opt(TT_KERNEL_TILE, std::max(2, bi / W), std::max(2, bo / W), 0, 0, 0);
                o.sd_vmax = 8192;
                vars.push_back(o);
            }

    // the heuristic tile on the slot-dim map with a cp.async ring of 3 or 4
    // stages (tile_sd_async_kernel): mixed on the suites, up to 1.18x on
    // latency-bound 4-byte gathers (profiles/round1_ab_sd_async.txt)
    if (hp.n >= 2 && hp.p[0] != 0)
        for (int st : {3, 4}) {
            tt_plan_options_t o = opt(TT_KERNEL_TILE, 0, 0, 0, 0, 0);
            o.slot_dims = 1;
            o.stages = st;
            vars.push_back(o);
        }

    // the heuristic tile with the vector-gather load phase (16-byte chunks of
    // the aligned superset of every input run, 3- or 4-stage cp.async ring),
    // and vector-gather tiles of shorter input / longer output runs (with
    // 16-byte chunk loads, short input runs cost little; the worst-case sweep
    // found its best tiles there: profiles/round2_vg_tile_sweep_worst12.jsonl)
    if (hp.n >= 2) {
        for (int st : {4, 3}) {
            tt_plan_options_t o = opt(TT_KERNEL_TILE, 0, 0, 0, 0, 0);
            o.vector_gather = 1;
            o.stages = st;
            vars.push_back(o);
        }
        for (int bi : {64, 128, 256})
            for (int bo : {256, 512, 1024, 2048}) {
                tt_plan_options_t o = opt(TT_KERNEL_TILE, std::max(2, bi / W), std::max(2, bo / W), 0, 0, 0);
                o.vector_gather = 1;
                o.stages = 3;
                vars.push_back(o);
            }
    }

    // the TMA-staged 2-D kernel where its strides allow (on plain 2-D
    // transposes it measured 0.90-0.95x of the vector 2-D kernel, but won on
    // some batched shapes: profiles/round2_ab_tma.jsonl)
    if (hp.n >= 2 && hp.p[0] != 0)
        for (int cps : {0, 2}) {
            tt_plan_options_t o = opt(0, 0, 0, 0, cps, 0);
            o.tma = 1;
            vars.push_back(o);
        }

    std::vector<Plan*> cands{heur};
    std::vector<std::string> keys{describe_json(*heur)};
    for (const auto& o : vars) {
        if (max_candidates > 0 && (int)cands.size() >= max_candidates) break;
        Plan* c = nullptr;
        if (create_plan_w(&c, rank, dims, perm, elem_size, stream, dev, &o, &cuda_occupancy, true) !=
            TT_SUCCESS)
            continue;
        std::string k = describe_json(*c);
        bool dup = false;
        for (const auto& kk : keys) dup |= kk == k;
        if (dup) { destroy_plan(c); continue; }
        cands.push_back(c);
        keys.push_back(k);
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        cudaGetLastError();
        for (Plan* c : cands) destroy_plan(c);
        return TT_CUDA_ERROR;
    }
    int best = 0;
    float bestMs = 1e30f, heurMs = 0.f;
    for (size_t i = 0; i < cands.size(); ++i) {
        // one timed launch first: a candidate over 4x the heuristic's time
        // is dropped without further repetitions
        cudaEventRecord(e0, s);
        if (launch_plan(*cands[i], in, out, stream) != 0) { cudaGetLastError(); continue; }
        cudaEventRecord(e1, s);
        if (cudaEventSynchronize(e1) != cudaSuccess) { cudaGetLastError(); continue; }
        if (i > 0) {
            float first = 0.f;
            cudaEventElapsedTime(&first, e0, e1);
            if (first > 4.f * heurMs) continue;
        }
        cudaEventRecord(e0, s);
        const int reps = 3;
        for (int r = 0; r < reps; ++r) launch_plan(*cands[i], in, out, stream);
        cudaEventRecord(e1, s);
        if (cudaEventSynchronize(e1) != cudaSuccess) { cudaGetLastError(); continue; }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        if (i == 0) heurMs = ms;
        if (ms < bestMs) { bestMs = ms; best = (int)i; }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (size_t i = 0; i < cands.size(); ++i)
        if ((int)i != best) destroy_plan(cands[i]);
    Plan* p = cands[best];
    p->measured = true;
    p->measured_ms = bestMs;
    p->heuristic_ms = heurMs;
    p->n_candidates = (int)cands.size();
    *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return TT_SUCCESS;
}

tt_status_t tt_plan_offline(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, const tt_device_props_t* props,
                            const tt_plan_options_t* opts) {
    DeviceInfo dev;
    dev.device = -1;
    if (props) {
        if (props->num_sms > 0) dev.num_sms = props->num_sms;
        if (props->max_smem_per_block > 0) dev.max_smem_per_block = props->max_smem_per_block;
        if (props->max_smem_per_sm > 0) dev.max_smem_per_sm = props->max_smem_per_sm;
        if (props->max_threads_per_sm > 0) dev.max_threads_per_sm = props->max_threads_per_sm;
        if (props->regs_per_sm > 0) dev.regs_per_sm = props->regs_per_sm;
    }
    return make_plan(plan, rank, dims, perm, elem_size, nullptr, dev, opts, nullptr);
}

static void props_to_dev(const tt_device_props_t* props, DeviceInfo& dev) {
    dev.device = -1;
    if (!props) return;
    if (props->num_sms > 0) dev.num_sms = props->num_sms;
    if (props->max_smem_per_block > 0) dev.max_smem_per_block = props->max_smem_per_block;
    if (props->max_smem_per_sm > 0) dev.max_smem_per_sm = props->max_smem_per_sm;
    if (props->max_threads_per_sm > 0) dev.max_threads_per_sm = props->max_threads_per_sm;
    if (props->regs_per_sm > 0) dev.regs_per_sm = props->regs_per_sm;
}

tt_status_t tt_plan_strided(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                            size_t elem_size, const int64_t* in_strides, const int64_t* out_strides,
                            tt_stream_t stream) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    tt_status_t st = validate(rank, dims, perm, elem_size);
    if (st != TT_SUCCESS) return st;
    DeviceInfo dev;
    st = query_device(dev);
    if (st != TT_SUCCESS) return st;
    Plan* p = nullptr;
    st = create_plan_s(&p, rank, dims, perm, elem_size, stream, dev, nullptr, &cuda_occupancy,
                       in_strides, out_strides);
    *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return st;
}

tt_status_t tt_plan_strided_offline(tt_plan_t* plan, int rank, const int64_t* dims, const int* perm,
                                    size_t elem_size, const int64_t* in_strides,
                                    const int64_t* out_strides, const tt_device_props_t* props,
                                    const tt_plan_options_t* opts) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    DeviceInfo dev;
    props_to_dev(props, dev);
    Plan* p = nullptr;
    tt_status_t st = create_plan_s(&p, rank, dims, perm, elem_size, nullptr, dev, opts, nullptr,
                                   in_strides, out_strides);
    *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return st;
}

tt_status_t tt_execute(tt_plan_t plan, const void* in, void* out) {
    NvtxRange nv("tt_execute");
    Plan* p = as_plan(plan);
    tt_status_t st = check_exec(p, in, out);
    if (st != TT_SUCCESS) return st;
    if (p->shard) return TT_INVALID_PLAN;  // sharded plans use tt_execute_sharded
    if (p->kc.acc) return TT_INVALID_PLAN;  // accumulate plans use tt_execute_scaled
    int e = launch_plan(*p, in, out, p->stream);
    return e == 0 ? TT_SUCCESS : TT_CUDA_ERROR;
}

tt_status_t tt_execute_scaled(tt_plan_t plan, const void* in, void* out, double alpha, double beta) {
    Plan* p = as_plan(plan);
    tt_status_t st = check_exec(p, in, out);
    if (st != TT_SUCCESS) return st;
    if (p->shard || !p->kc.acc) return TT_INVALID_PLAN;
    int e = launch_plan_scaled(*p, in, out, p->stream, alpha, beta);
    return e == 0 ? TT_SUCCESS : TT_CUDA_ERROR;
}

tt_status_t tt_execute_host(tt_plan_t plan, const void* host_in, void* host_out, void* dev_in,
                            void* dev_out) {
    Plan* p = as_plan(plan);
    if (p == nullptr) return TT_INVALID_PLAN;
    if (host_in == nullptr || host_out == nullptr) return TT_INVALID_PARAMETER;
    tt_status_t st = check_exec(p, dev_in, dev_out);
    if (st != TT_SUCCESS) return st;
    if (p->shard) return TT_INVALID_PLAN;
    if (!p->prob.dense) return TT_UNSUPPORTED;  // host path: dense tensors only
    const size_t bytes = (size_t)p->prob.vol * (size_t)p->prob.esize;
    cudaStream_t s = static_cast<cudaStream_t>(p->stream);
    if (bytes >= kPipeMinBytes) {
        st = execute_host_pipelined(*p, host_in, host_out, dev_in, dev_out);
        if (st != TT_UNSUPPORTED) return st;
    }
    if (cudaMemcpyAsync(dev_in, host_in, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    if (launch_plan(*p, dev_in, dev_out, p->stream) != 0) return TT_CUDA_ERROR;
    if (cudaMemcpyAsync(host_out, dev_out, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    return TT_SUCCESS;
}

tt_status_t tt_plan_describe(tt_plan_t plan, char* buf, size_t len) {
    Plan* p = as_plan(plan);
    if (p == nullptr) return TT_INVALID_PLAN;
    if (buf == nullptr || len == 0) return TT_INVALID_PARAMETER;
    std::string s = p->shard ? describe_shard_json(*p) : describe_json(*p);
    if (s.size() + 1 > len) {
        std::memcpy(buf, s.data(), len - 1);
        buf[len - 1] = '\0';
        return TT_BUFFER_TOO_SMALL;
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return TT_SUCCESS;
}

int tt_plan_launches(tt_plan_t plan) {
    Plan* p = as_plan(plan);
    if (p == nullptr) return -1;
    if (p->shard) return shard_launches(p->shard);
    return 1;
}

tt_status_t tt_destroy(tt_plan_t plan) {
    if (!retire_handle(plan)) return TT_INVALID_PLAN;  // NULL, never issued, or already destroyed
    destroy_plan(reinterpret_cast<Plan*>(plan));
    return TT_SUCCESS;
}

}  // extern "C"
