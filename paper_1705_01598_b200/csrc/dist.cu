// dist.cu -- sharded permutation over the GPUs of one box (row e).
//
// The paper has no multi-GPU transpose ("we will only consider local
// tensor transposes"); this is the BASELINE.json north_star extension:
//
//   global dims D[0..n-1], perm p, P ranks.  Input block-sharded along input
//   dim n-1 (rank r holds D[n-1]/P of it), output block-sharded along output
//   dim n-1 = input dim t = p[n-1].
//
//   t == n-1  "local":       each rank permutes its slab with p; no traffic.
//   t != n-1  "redistribute": pack  = local permute of the slab into output
//                             order with dim t split (D[t]/P inner, P outer)
//                             and the P part outermost, so the block for
//                             destination q is contiguous;
//                             ncclAlltoAll over NVLink 5 / NVSwitch;
//                             unpack = (inner, middle, P) -> (inner, P, middle)
//                             moving the source rank next to the output
//                             position j* of input dim n-1 (p[j*] = n-1).
//
//   t != n-1  "p2p" (SURVEY f-1, fused): no pack, no NCCL copy, no unpack.
//             Rank r's slab splits along input dim t into P sub-boxes
//             x_t in [q*c, (q+1)*c), c = D[t]/P; sub-box q lands in output
//             slab q (on rank q's GPU) as a contiguous range of output dim
//             j* (p[j*] = n-1), at y_{j*} = r*D[n-1]/P + x_{n-1}.  All P
//             sub-boxes share ONE strided plan (tt_plan_strided geometry):
//             extents = slab with dim t cut to c, input strides = the slab's,
//             output strides = the output slab's; only the base pointers
//             differ: in + q*c*S_in[t], out_q + r*(D[n-1]/P)*S_out[j*].
//             The permute kernel stores straight into the peers' output
//             slabs over NVLink (CUDA IPC mappings), so HBM traffic is the
//             2S minimum and the transfer overlaps the permutation tile by
//             tile.  Two device-side barriers over IPC-mapped signal words
//             (entry: peers are done with their output slabs; exit: all
//             stores into mine have landed) replace the collective.
//
// All local steps are ordinary single-GPU plans (planner.cpp + kernels.cu).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "tt_internal.h"

namespace tt {

static int64_t ceil_div_i64(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct tt_comm_impl {
    ncclComm_t nccl = nullptr;
    int nranks = 0, rank = 0, device = -1;
};

struct ShardInfo {
    tt_comm_impl* comm = nullptr;   // null for offline plans
    int nranks = 1, rank = 0;
    bool redistribute = false;
    Plan* local = nullptr;          // local mode
    Plan* pack = nullptr;           // redistribute mode
    Plan* unpack = nullptr;
    void* send = nullptr;           // staging, shard bytes each
    void* recv = nullptr;
    size_t shard_bytes = 0;
    size_t a2a_count = 0;           // elements per peer
    int esize = 4;
    std::vector<int64_t> local_in, local_out;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool timed = false;
    // chunked exchange (redistribute mode, chunks > 1): the split dim t's
    // per-destination extent c is cut into chunks of ct (the last one
    // ctail); pack / all-to-all / unpack of chunk k overlap those of k+-1
    int chunks = 1;
    int64_t ct = 0, ctail = 0;
    int64_t w = 0;                  // elements per destination per unit of t
    int64_t sinT = 0;               // slab stride of input dim t (elements)
    Plan* pack_tail = nullptr;      // plans of the last chunk when ctail != ct
    Plan* unpack_tail = nullptr;
    cudaStream_t cstream = nullptr; // all-to-all (high priority)
    cudaStream_t ustream = nullptr; // unpack
    std::vector<cudaEvent_t> evPack, evA2a;
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    cudaEvent_t evT[4] = {nullptr, nullptr, nullptr, nullptr};  // a2a start/end, unpack start/end
    // p2p mode (f-1)
    bool p2p = false;
    int proc = 0;                   // this process's slab index
    Plan* fused = nullptr;          // one strided plan for every destination sub-box
    int64_t in_step = 0;            // elements between destination sub-boxes in the input slab
    int64_t out_off = 0;            // this rank's block inside every output slab (elements)
    void* reg_out = nullptr;        // registered output slab (tt_sharded_register_output)
    void* exported = nullptr;       // output slab of tt_sharded_export_record, until imported
    std::vector<void*> peer_out;    // [P] output slabs as mapped in this process
    std::vector<void*> ipc_bases;   // peer allocations opened with cudaIpcOpenMemHandle
    int* sig = nullptr;             // [P] signal words of this rank (device), + [P] error word
    std::vector<int*> peer_sig;     // [P] peers' signal arrays as mapped here
    int epoch = 0;
    // the P sub-box launches run concurrently on P streams forked from the
    // plan's stream, each with 1/P of the plan's persistent grid: together
    // they sweep the input slab densely (one launch per destination after
    // another would read it P times at 1/P density -- measured 3-8x slower)
    std::vector<cudaStream_t> sub;
    std::vector<cudaEvent_t> join;
    cudaEvent_t fork = nullptr;
};

void destroy_shard(ShardInfo* s) {
    if (!s) return;
    destroy_plan(s->local);
    destroy_plan(s->pack);
    destroy_plan(s->unpack);
    destroy_plan(s->fused);
    destroy_plan(s->pack_tail);
    destroy_plan(s->unpack_tail);
    if (s->cstream) cudaStreamDestroy(s->cstream);
    if (s->ustream) cudaStreamDestroy(s->ustream);
    for (cudaEvent_t e : s->evPack) cudaEventDestroy(e);
    for (cudaEvent_t e : s->evA2a) cudaEventDestroy(e);
    if (s->evFork) cudaEventDestroy(s->evFork);
    if (s->evJoin) cudaEventDestroy(s->evJoin);
    for (auto& e : s->evT)
        if (e) cudaEventDestroy(e);
    for (void* b : s->ipc_bases) cudaIpcCloseMemHandle(b);
    if (s->sig) cudaFree(s->sig);
    for (cudaStream_t x : s->sub) cudaStreamDestroy(x);
    for (cudaEvent_t e : s->join) cudaEventDestroy(e);
    if (s->fork) cudaEventDestroy(s->fork);
    if (s->send) cudaFree(s->send);
    if (s->recv) cudaFree(s->recv);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    delete s;
}

int shard_launches(const ShardInfo* s) {
    if (!s->redistribute) return 1;
    if (s->p2p) return s->nranks + (s->comm ? 2 : 0);  // P sub-box launches (+ 2 barriers)
    return s->chunks * (s->nranks > 1 ? 3 : 2);  // per chunk: pack, (NCCL all-to-all), unpack
}

std::string describe_shard_json(const Plan& plan) {
    const ShardInfo* s = plan.shard;
    std::ostringstream o;
    auto arr = [&](const std::vector<int64_t>& v) {
        o << "[";
        for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << (long long)v[i];
        o << "]";
    };
    o << "{\"version\":" << TT_VERSION << ",\"sharded\":true,\"nranks\":" << s->nranks
      << ",\"rank\":" << s->rank << ",\"mode\":\""
      << (s->redistribute ? (s->p2p ? "p2p" : "redistribute") : "local")
      << "\",\"elem_size\":" << s->esize << ",\"global_dims\":";
    arr(plan.dims);
    o << ",\"perm\":[";
    for (int i = 0; i < plan.rank; ++i) o << (i ? "," : "") << plan.perm[i];
    o << "],\"local_in_dims\":";
    arr(s->local_in);
    o << ",\"local_out_dims\":";
    arr(s->local_out);
    o << ",\"shard_bytes\":" << s->shard_bytes << ",\"a2a_count\":" << s->a2a_count
      << ",\"launches\":" << shard_launches(s);
    if (s->local) o << ",\"local\":" << describe_json(*s->local);
    if (s->redistribute && !s->p2p)
        o << ",\"chunks\":" << s->chunks << ",\"chunk_t\":" << (long long)s->ct
          << ",\"chunk_tail\":" << (long long)s->ctail << ",\"chunk_w\":" << (long long)s->w
          << ",\"chunk_in_step\":" << (long long)s->sinT;
    if (s->pack) o << ",\"pack\":" << describe_json(*s->pack);
    if (s->unpack) o << ",\"unpack\":" << describe_json(*s->unpack);
    if (s->pack_tail) o << ",\"pack_tail\":" << describe_json(*s->pack_tail);
    if (s->unpack_tail) o << ",\"unpack_tail\":" << describe_json(*s->unpack_tail);
    if (s->fused) {
        o << ",\"in_step\":" << (long long)s->in_step << ",\"out_offset\":" << (long long)s->out_off
          << ",\"dest_order\":[";
        for (int k = 1; k <= s->nranks; ++k) o << (k > 1 ? "," : "") << (s->proc + k) % s->nranks;
        o << "],\"fused\":" << describe_json(*s->fused);
    }
    o << "}";
    return o.str();
}

// Geometry + sub-plans; comm may be null (offline).
static tt_status_t build_shard_n(Plan** out, tt_comm_impl* comm, int nranks, int rank, int n,
                                 const int64_t* gd, const int* perm, size_t esize, void* stream,
                                 const DeviceInfo& dev, OccupancyFn occ, bool p2p = false,
                                 bool forceRedist = false, int chunksOpt = 0) {
    *out = nullptr;
    tt_status_t st = validate(n, gd, perm, esize);
    if (st != TT_SUCCESS) return st;
    if (nranks < 1 || rank < 0 || rank >= nranks) return TT_INVALID_PARAMETER;
    const int P = nranks;
    const int t = perm[n - 1];
    if (gd[n - 1] % P != 0) return TT_UNSUPPORTED;
    // forceRedist (option force_redistribute, tests): take the redistribution
    // path even with one rank, so the NCCL / P2P machinery runs on one GPU
    const bool redist = (t != n - 1) && (P > 1 || forceRedist);
    if (redist && gd[t] % P != 0) return TT_UNSUPPORTED;

    ShardInfo* s = new (std::nothrow) ShardInfo();
    Plan* outer = new (std::nothrow) Plan();
    if (!s || !outer) { delete s; delete outer; return TT_INTERNAL_ERROR; }
    s->comm = comm;
    s->nranks = P;
    s->rank = rank;
    s->esize = (int)esize;
    s->redistribute = redist;
    s->proc = rank;
    s->p2p = redist && p2p;
    outer->device = dev.device;
    outer->stream = stream;
    outer->rank = n;
    outer->dims.assign(gd, gd + n);
    outer->perm.assign(perm, perm + n);
    outer->prob = normalize(n, gd, perm, (int)esize, true);
    outer->shard = s;

    std::vector<int64_t> L(gd, gd + n);
    L[n - 1] /= P;
    s->local_in = L;
    int64_t shard_vol = 1;
    for (int64_t x : L) shard_vol *= x;
    s->shard_bytes = (size_t)shard_vol * esize;
    s->local_out.resize(n);
    for (int j = 0; j < n; ++j) s->local_out[j] = gd[perm[j]];
    s->local_out[n - 1] /= P;  // output dim n-1 is input dim t, sharded

    if (!redist) {
        // local: output slab r = permute(input slab r) (t == n-1 or P == 1)
        std::vector<int64_t> ld = L;
        if (P == 1) ld[n - 1] = gd[n - 1];
        st = create_plan(&s->local, n, ld.data(), perm, esize, stream, dev, nullptr, occ);
        if (st != TT_SUCCESS) { destroy_plan(outer); return st; }
        *out = outer;
        return TT_SUCCESS;
    }

    const int64_t c = gd[t] / P;
    if (s->p2p) {
        // fused: one strided plan per destination sub-box (x_t in [q*c, (q+1)*c))
        std::vector<int64_t> fd = L, si(n), so(n);
        fd[t] = c;
        int64_t acc = 1;
        for (int i = 0; i < n; ++i) { si[i] = acc; acc *= L[i]; }  // the slab's strides
        acc = 1;
        int jstar = -1;
        for (int j = 0; j < n; ++j) {                              // the output slab's strides
            so[j] = acc;
            acc *= s->local_out[j];
            if (perm[j] == n - 1) jstar = j;
        }
        s->in_step = c * si[t];
        s->out_off = (int64_t)rank * L[n - 1] * so[jstar];
        st = create_plan_s(&s->fused, n, fd.data(), perm, esize, stream, dev, nullptr, occ,
                           si.data(), so.data());
        if (st != TT_SUCCESS) { destroy_plan(outer); return st; }
        // the P sub-box launches run concurrently (launch_fused): 1/P of the grid each
        KernelChoice& kc = s->fused->kc;
        kc.grid = (int)std::max<int64_t>(1, ceil_div_i64(kc.grid, P));
        kc.fb_grid = (int)std::max<int64_t>(1, ceil_div_i64(kc.fb_grid, P));
        *out = outer;
        return TT_SUCCESS;
    }

    // chunks of the exchange along t (per destination: c -> K chunks of ct,
    // the last ctail): default 4 from 32 MB of shard (below that the extra
    // launches and all-to-alls cost more than the overlap wins)
    int K = chunksOpt > 0 ? chunksOpt : (s->shard_bytes >= (size_t(32) << 20) ? 4 : 1);
    if (K > c) K = (int)c;
    s->ct = ceil_div_i64(c, K);
    s->chunks = (int)ceil_div_i64(c, s->ct);
    s->ctail = c - (int64_t)(s->chunks - 1) * s->ct;
    s->w = shard_vol / L[t];
    {
        int64_t acc = 1;
        for (int i = 0; i < t; ++i) acc *= L[i];
        s->sinT = acc;
    }

    // pack: split input dim t into (e, P) -- e = c, or a chunk's extent --
    // P-part outermost, so the block for destination q is contiguous.
    // Unchunked: a dense problem; chunk k: the sub-box x_t in
    // q*c + k*ct + [0, e) of every destination q, input strides of the slab
    // (the P part steps c * S_t), base offset k*ct*S_t (launch time).
    auto ni = [&](int i) { return i < t ? i : (i == t ? t : i + 1); };
    std::vector<int> pp;
    for (int j = 0; j < n; ++j) pp.push_back(ni(perm[j]));
    pp.push_back(t + 1);
    auto make_pack = [&](int64_t e, Plan** dst) {
        std::vector<int64_t> pd, ps;
        int64_t acc = 1;
        for (int i = 0; i < n; ++i) {
            if (i == t) {
                pd.push_back(e); ps.push_back(acc);
                pd.push_back(P); ps.push_back(acc * c);
            } else {
                pd.push_back(L[i]); ps.push_back(acc);
            }
            acc *= L[i];
        }
        if (s->chunks == 1)
            return create_plan(dst, n + 1, pd.data(), pp.data(), esize, stream, dev, nullptr, occ);
        return create_plan_s(dst, n + 1, pd.data(), pp.data(), esize, stream, dev, nullptr, occ, ps.data(),
                             nullptr);
    };
    st = make_pack(s->chunks == 1 ? c : s->ct, &s->pack);
    if (st == TT_SUCCESS && s->chunks > 1 && s->ctail != s->ct) st = make_pack(s->ctail, &s->pack_tail);
    if (st != TT_SUCCESS) { destroy_plan(outer); return st; }

    // unpack: received [e'_0 .. e'_{n-1}, P_src] -> move P_src after j*
    // (chunk k: e'_{n-1} is the chunk's extent; its output is the contiguous
    // range of output dim n-1 starting at k*ct)
    int jstar = -1;
    for (int j = 0; j < n; ++j)
        if (perm[j] == n - 1) jstar = j;
    auto make_unpack = [&](int64_t e, Plan** dst) {
        int64_t inner = 1, middle = 1;
        for (int j = 0; j < n; ++j) {
            const int64_t ej = (j == n - 1) ? e : L[perm[j]];
            if (j <= jstar) inner *= ej;
            else middle *= ej;
        }
        const int64_t ud[3] = {inner, middle, (int64_t)P};
        const int up[3] = {0, 2, 1};
        return create_plan(dst, 3, ud, up, esize, stream, dev, nullptr, occ);
    };
    st = make_unpack(s->chunks == 1 ? c : s->ct, &s->unpack);
    if (st == TT_SUCCESS && s->chunks > 1 && s->ctail != s->ct) st = make_unpack(s->ctail, &s->unpack_tail);
    if (st != TT_SUCCESS) { destroy_plan(outer); return st; }
    s->a2a_count = (size_t)(shard_vol / P);
    *out = outer;
    return TT_SUCCESS;
}

// ---- p2p (f-1): device-side barrier over IPC-mapped signal words ----------
//
// Rank r's signal array sig[0..P-1] (+ one error word at sig[P]) lives in its
// own HBM; peer q writes sig[q] = epoch when it arrives.  Thread q of the
// barrier kernel publishes this rank's arrival in peer q's array with a
// system-scope release store and then waits, with system-scope acquire loads,
// until peer q's word in its own array reaches the epoch.  The fence before the
// release makes every store this rank issued earlier on the stream (the fused
// permute kernels writing into peers' slabs over NVLink) visible first.  A
// peer that never arrives sets the error word after kP2PTimeoutNs instead of
// hanging the GPU (reported by tt_sharded_timings).
constexpr int kMaxPeers = 64;
constexpr unsigned long long kP2PTimeoutNs = 30ull * 1000 * 1000 * 1000;

struct BarrierArgs {
    int* peer_sig[kMaxPeers];
    int* mine;
    int P, rank, epoch;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void p2p_barrier_kernel(const __grid_constant__ BarrierArgs a) {
    const int q = threadIdx.x;
    if (q >= a.P) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(a.peer_sig[q] + a.rank), "r"(a.epoch)
                 : "memory");
    const unsigned long long t0 = global_ns();
    for (;;) {
        int v;
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(a.mine + q) : "memory");
        if (v - a.epoch >= 0) break;
        if (global_ns() - t0 > kP2PTimeoutNs) {
            // a peer is missing: record it and stop the stream for good (the
            // context's sticky launch error makes every later tt_* call and
            // synchronisation fail) -- never let the fused stores run into
            // slabs a peer may still be reading, or hand out a slab whose
            // peers' stores have not landed
            atomicExch(a.mine + a.P, 1);
            __threadfence_system();
            __trap();
        }
        __nanosleep(200);
    }
}

// Chunked exchange: chunk k = x_t in q*c + k*ct + [0, e_k) for every
// destination q.  Its pack (plan stream) fills send[k*P*w*ct ..) as P
// contiguous blocks of w*e_k words; its all-to-all (cstream) waits for that
// pack; its unpack (ustream) waits for that all-to-all and writes output
// slab range k*ct*w*P (output dim n-1 from k*ct).  The buffers are reused
// by the next execute only after the plan stream joined the last unpack.
static tt_status_t execute_chunked(ShardInfo* s, const void* in, void* out, cudaStream_t st) {
    const int P = s->nranks, K = s->chunks;
    const size_t E = (size_t)s->esize;
    const ncclDataType_t dt = s->esize == 4 ? ncclUint32 : ncclUint64;
    const char* ib = static_cast<const char*>(in);
    char* ob = static_cast<char*>(out);
    char* sb = static_cast<char*>(s->send);
    char* rb = static_cast<char*>(s->recv);
    NvtxRange nv("tt_execute_sharded chunked (pack | all-to-all | unpack)");
    if (cudaEventRecord(s->ev[0], st) != cudaSuccess || cudaEventRecord(s->evFork, st) != cudaSuccess ||
        cudaStreamWaitEvent(s->cstream, s->evFork, 0) != cudaSuccess ||
        cudaStreamWaitEvent(s->ustream, s->evFork, 0) != cudaSuccess)
        return TT_CUDA_ERROR;
    for (int k = 0; k < K; ++k) {
        const bool tail = k == K - 1 && s->pack_tail != nullptr;
        const int64_t e = k == K - 1 ? s->ctail : s->ct;
        const size_t blk = (size_t)k * (size_t)s->ct;  // t offset of the chunk
        const size_t off = blk * (size_t)s->w * (size_t)P * E;
        if (launch_plan(tail ? *s->pack_tail : *s->pack, ib + blk * (size_t)s->sinT * E, sb + off, st) != 0)
            return TT_CUDA_ERROR;
        if (cudaEventRecord(s->evPack[k], st) != cudaSuccess ||
            cudaStreamWaitEvent(s->cstream, s->evPack[k], 0) != cudaSuccess)
            return TT_CUDA_ERROR;
        if (k == 0 && cudaEventRecord(s->evT[0], s->cstream) != cudaSuccess) return TT_CUDA_ERROR;
        if (ncclAlltoAll(sb + off, rb + off, (size_t)s->w * (size_t)e, dt, s->comm->nccl, s->cstream) !=
            ncclSuccess)
            return TT_NCCL_ERROR;
        if (cudaEventRecord(s->evA2a[k], s->cstream) != cudaSuccess ||
            cudaStreamWaitEvent(s->ustream, s->evA2a[k], 0) != cudaSuccess)
            return TT_CUDA_ERROR;
        if (k == 0 && cudaEventRecord(s->evT[2], s->ustream) != cudaSuccess) return TT_CUDA_ERROR;
        if (launch_plan(tail ? *s->unpack_tail : *s->unpack, rb + off, ob + off, s->ustream) != 0)
            return TT_CUDA_ERROR;
    }
    if (cudaEventRecord(s->ev[1], st) != cudaSuccess || cudaEventRecord(s->evT[1], s->cstream) != cudaSuccess ||
        cudaEventRecord(s->evT[3], s->ustream) != cudaSuccess ||
        cudaEventRecord(s->evJoin, s->ustream) != cudaSuccess || cudaStreamWaitEvent(st, s->evJoin, 0) != cudaSuccess ||
        cudaEventRecord(s->ev[3], st) != cudaSuccess)
        return TT_CUDA_ERROR;
    s->timed = true;
    return TT_SUCCESS;
}

static int launch_barrier(ShardInfo* s, cudaStream_t st, int epoch) {
    BarrierArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int q = 0; q < s->nranks; ++q) a.peer_sig[q] = s->peer_sig[q];
    a.mine = s->sig;
    a.P = s->nranks;
    a.rank = s->proc;
    a.epoch = epoch;
    p2p_barrier_kernel<<<1, 64, 0, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// The P sub-box permutations of one fused execute, nearest-rank-last order
// (destination proc+1 first, own slab last) so that at any moment the ranks
// write to different peers.
static tt_status_t launch_fused(ShardInfo* s, const void* in, void* const* outs, void* stream) {
    const int P = s->nranks;
    cudaStream_t main = static_cast<cudaStream_t>(stream);
    if (P > 1 && s->sub.empty()) {  // first execute: fork/join streams and events
        s->sub.assign(P, nullptr);
        s->join.assign(P, nullptr);
        bool ok = cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming) == cudaSuccess;
        for (int q = 0; q < P && ok; ++q)
            ok = cudaStreamCreateWithFlags(&s->sub[q], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&s->join[q], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) { cudaGetLastError(); return TT_CUDA_ERROR; }
    }
    if (P > 1 && cudaEventRecord(s->fork, main) != cudaSuccess) return TT_CUDA_ERROR;
    const char* ib = static_cast<const char*>(in);
    for (int k = 1; k <= P; ++k) {
        const int q = (s->proc + k) % P;
        const void* i = ib + (size_t)q * (size_t)s->in_step * s->esize;
        void* o = static_cast<char*>(outs[q]) + (size_t)s->out_off * s->esize;
        cudaStream_t x = P > 1 ? s->sub[q] : main;
        if (P > 1 && cudaStreamWaitEvent(x, s->fork, 0) != cudaSuccess) return TT_CUDA_ERROR;
        if (launch_plan(*s->fused, i, o, x) != 0) return TT_CUDA_ERROR;
        if (P > 1 && cudaEventRecord(s->join[q], x) != cudaSuccess) return TT_CUDA_ERROR;
    }
    for (int q = 0; q < P && P > 1; ++q)
        if (cudaStreamWaitEvent(main, s->join[q], 0) != cudaSuccess) return TT_CUDA_ERROR;
    return TT_SUCCESS;
}

// Base and offset of a device pointer inside its allocation (for CUDA IPC,
// whose handles name whole allocations).  Driver entry point, so libtt does
// not link libcuda directly.
typedef CUresult (*MemRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
static bool alloc_base(const void* p, void** base, size_t* off) {
    static MemRangeFn fn = nullptr;
    if (fn == nullptr) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault,
                                             &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || f == nullptr) {
            cudaGetLastError();
            return false;
        }
        fn = reinterpret_cast<MemRangeFn>(f);
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
    *base = reinterpret_cast<void*>(b);
    *off = reinterpret_cast<uintptr_t>(p) - (uintptr_t)b;
    return true;
}

// What each rank contributes to the registration all-gather.
struct RegRecord {
    cudaIpcMemHandle_t out;
    cudaIpcMemHandle_t sig;
    int64_t out_off;
    int32_t device, proc;
    int32_t ok;        // 1: this rank's handles are valid (a failed rank still joins the exchange)
    char pad[256 - 2 * sizeof(cudaIpcMemHandle_t) - 20];
};
static_assert(sizeof(RegRecord) == TT_SHARD_RECORD_BYTES, "registration record");

// This rank's record: its signal words (allocated once, zeroed, reused on a
// retry) and the IPC handles of the allocations holding them and out_local.
static tt_status_t make_record(ShardInfo* s, int device, void* out_local, RegRecord& mine) {
    std::memset(&mine, 0, sizeof(mine));
    mine.device = device;
    mine.proc = s->proc;
    const int P = s->nranks;
    if (s->sig == nullptr && cudaMalloc(&s->sig, (P + 1) * sizeof(int)) != cudaSuccess) {
        s->sig = nullptr;
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    if (cudaMemset(s->sig, 0, (P + 1) * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    void* base = nullptr;
    size_t off = 0;
    if (!alloc_base(out_local, &base, &off) || cudaIpcGetMemHandle(&mine.out, base) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.sig, s->sig) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    mine.out_off = (int64_t)off;
    mine.ok = 1;
    return TT_SUCCESS;
}

// Open every peer's record (all[q] is rank q's); on any failure nothing stays open.
static tt_status_t open_records(ShardInfo* s, void* out_local, const RegRecord* all) {
    const int P = s->nranks;
    for (int q = 0; q < P; ++q)
        if (!all[q].ok || all[q].proc != q) return TT_INVALID_PARAMETER;
    std::vector<void*> opened;
    std::vector<void*> pout(P, nullptr);
    std::vector<int*> psig(P, nullptr);
    for (int q = 0; q < P; ++q) {
        if (q == s->proc) {
            pout[q] = out_local;
            psig[q] = s->sig;
            continue;
        }
        void* ob = nullptr;
        void* sb = nullptr;
        if (cudaIpcOpenMemHandle(&ob, all[q].out, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess)
            opened.push_back(ob);
        else
            ob = nullptr;
        if (ob && cudaIpcOpenMemHandle(&sb, all[q].sig, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess)
            opened.push_back(sb);
        else
            sb = nullptr;
        if (!ob || !sb) {
            cudaGetLastError();
            for (void* b : opened) cudaIpcCloseMemHandle(b);
            return TT_CUDA_ERROR;
        }
        pout[q] = static_cast<char*>(ob) + all[q].out_off;
        psig[q] = static_cast<int*>(sb);
    }
    s->ipc_bases = opened;
    s->peer_out = pout;
    s->peer_sig = psig;
    s->reg_out = out_local;
    return TT_SUCCESS;
}

}  // namespace tt

using namespace tt;

static tt_comm_impl* as_comm(tt_comm_t c) {
    return handle_live(c) ? reinterpret_cast<tt_comm_impl*>(c) : nullptr;
}

extern "C" {

tt_status_t tt_comm_unique_id(void* id) {
    if (id == nullptr) return TT_INVALID_PARAMETER;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return TT_NCCL_ERROR;
    static_assert(sizeof(u) == TT_NCCL_UNIQUE_ID_BYTES, "unique id size");
    std::memcpy(id, &u, sizeof(u));
    return TT_SUCCESS;
}

tt_status_t tt_comm_init(tt_comm_t* comm, const void* id, int nranks, int rank) {
    if (comm == nullptr || id == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
        return TT_INVALID_PARAMETER;
    *comm = nullptr;
    tt_comm_impl* c = new (std::nothrow) tt_comm_impl();
    if (!c) return TT_INTERNAL_ERROR;
    if (cudaGetDevice(&c->device) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return TT_INVALID_DEVICE;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    if (ncclCommInitRank(&c->nccl, nranks, u, rank) != ncclSuccess) {
        delete c;
        return TT_NCCL_ERROR;
    }
    c->nranks = nranks;
    c->rank = rank;
    *comm = reinterpret_cast<tt_comm_t>(publish_handle(c));
    return TT_SUCCESS;
}

tt_status_t tt_comm_destroy(tt_comm_t comm) {
    if (!retire_handle(comm)) return TT_INVALID_PARAMETER;  // NULL or already destroyed
    tt_comm_impl* c = reinterpret_cast<tt_comm_impl*>(comm);
    ncclResult_t r = ncclCommDestroy(c->nccl);
    delete c;
    return r == ncclSuccess ? TT_SUCCESS : TT_NCCL_ERROR;
}

tt_status_t tt_plan_sharded(tt_plan_t* plan, tt_comm_t comm, int ndims, const int64_t* global_dims,
                            const int* perm, size_t elem_size, tt_stream_t stream) {
    return tt_plan_sharded_ex(plan, comm, ndims, global_dims, perm, elem_size, stream, nullptr);
}

tt_status_t tt_plan_sharded_ex(tt_plan_t* plan, tt_comm_t comm, int ndims, const int64_t* global_dims,
                               const int* perm, size_t elem_size, tt_stream_t stream,
                               const tt_plan_options_t* opts) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    tt_comm_impl* c = as_comm(comm);
    if (c == nullptr) return TT_INVALID_PARAMETER;
    if (ndims < 1) return TT_INVALID_PARAMETER;
    const int rank = c->rank;
    DeviceInfo dev;
    tt_status_t st = query_device(dev);
    if (st != TT_SUCCESS) return st;
    if (dev.device != c->device) return TT_INVALID_DEVICE;
    Plan* p = nullptr;
    st = build_shard_n(&p, c, c->nranks, rank, ndims, global_dims, perm, elem_size, stream, dev,
                       &cuda_occupancy, false, opts && opts->force_redistribute, opts ? opts->a2a_chunks : 0);
    if (st != TT_SUCCESS) return st;
    ShardInfo* s = p->shard;
    if (s->redistribute) {
        if (cudaMalloc(&s->send, s->shard_bytes) != cudaSuccess ||
            cudaMalloc(&s->recv, s->shard_bytes) != cudaSuccess) {
            cudaGetLastError();
            destroy_plan(p);
            return TT_CUDA_ERROR;
        }
    }
    if (s->redistribute && s->chunks > 1) {
        // the exchange gets the highest stream priority: the pack and unpack
        // kernels' persistent grids must not keep NCCL's kernels off the SMs
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        bool ok = cudaStreamCreateWithPriority(&s->cstream, cudaStreamNonBlocking, hi) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&s->ustream, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&s->evFork, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&s->evJoin, cudaEventDisableTiming) == cudaSuccess;
        s->evPack.assign(s->chunks, nullptr);
        s->evA2a.assign(s->chunks, nullptr);
        for (int k = 0; k < s->chunks && ok; ++k)
            ok = cudaEventCreateWithFlags(&s->evPack[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&s->evA2a[k], cudaEventDisableTiming) == cudaSuccess;
        for (auto& e : s->evT)
            if (ok) ok = cudaEventCreate(&e) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            destroy_plan(p);
            return TT_CUDA_ERROR;
        }
    }
    for (auto& e : s->ev) {
        if (cudaEventCreate(&e) != cudaSuccess) {
            cudaGetLastError();
            destroy_plan(p);
            return TT_CUDA_ERROR;
        }
    }
    *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return TT_SUCCESS;
}

tt_status_t tt_plan_sharded_offline(tt_plan_t* plan, int nranks, int rank, int ndims,
                                    const int64_t* global_dims, const int* perm, size_t elem_size) {
    return tt_plan_sharded_offline_ex(plan, nranks, rank, ndims, global_dims, perm, elem_size, nullptr);
}

tt_status_t tt_plan_sharded_offline_ex(tt_plan_t* plan, int nranks, int rank, int ndims,
                                       const int64_t* global_dims, const int* perm, size_t elem_size,
                                       const tt_plan_options_t* opts) {
    if (ndims < 1) return TT_INVALID_PARAMETER;
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    DeviceInfo dev;
    dev.device = -1;
    Plan* p = nullptr;
    tt_status_t st = build_shard_n(&p, nullptr, nranks, rank, ndims, global_dims, perm, elem_size,
                                   nullptr, dev, nullptr, false, opts && opts->force_redistribute,
                                   opts ? opts->a2a_chunks : 0);
    if (st == TT_SUCCESS) *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return st;
}

tt_status_t tt_execute_sharded(tt_plan_t plan, const void* in_local, void* out_local) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    if (in_local == nullptr || out_local == nullptr || in_local == out_local)
        return TT_INVALID_PARAMETER;
    if (((reinterpret_cast<uintptr_t>(in_local) | reinterpret_cast<uintptr_t>(out_local)) &
         (uintptr_t)(s->esize - 1)) != 0)
        return TT_INVALID_PARAMETER;
    // a communicator, or a p2p plan registered through exported / imported records
    if ((s->comm == nullptr && !(s->p2p && s->reg_out != nullptr)) || p->device < 0) return TT_INVALID_DEVICE;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    if (!s->redistribute)
        return launch_plan(*s->local, in_local, out_local, p->stream) == 0 ? TT_SUCCESS : TT_CUDA_ERROR;
    if (s->p2p) {
        // fused: entry barrier, P sub-box permutations into the peers' slabs, exit barrier
        if (s->reg_out == nullptr || out_local != s->reg_out) return TT_INVALID_PARAMETER;
        // epochs advance by two per execute whatever happens below, so a
        // failed execute cannot leave this rank one barrier behind its peers
        const int base = s->epoch;
        s->epoch += 2;
        NvtxRange nv("tt_execute_sharded p2p (barrier, fused stores, barrier)");
        cudaEventRecord(s->ev[0], st);
        if (launch_barrier(s, st, base + 1) != 0) return TT_CUDA_ERROR;
        cudaEventRecord(s->ev[1], st);
        tt_status_t rc = launch_fused(s, in_local, s->peer_out.data(), p->stream);
        if (rc != TT_SUCCESS) return rc;
        cudaEventRecord(s->ev[2], st);
        if (launch_barrier(s, st, base + 2) != 0) return TT_CUDA_ERROR;
        cudaEventRecord(s->ev[3], st);
        s->timed = true;
        return TT_SUCCESS;
    }
    if (s->chunks > 1) return execute_chunked(s, in_local, out_local, st);
    cudaEventRecord(s->ev[0], st);
    {
        NvtxRange nv("tt_execute_sharded pack");
        if (launch_plan(*s->pack, in_local, s->send, p->stream) != 0) return TT_CUDA_ERROR;
    }
    cudaEventRecord(s->ev[1], st);
    const ncclDataType_t dt = s->esize == 4 ? ncclUint32 : ncclUint64;
    {
        NvtxRange nv("tt_execute_sharded all-to-all");
        if (ncclAlltoAll(s->send, s->recv, s->a2a_count, dt, s->comm->nccl, st) != ncclSuccess)
            return TT_NCCL_ERROR;
    }
    cudaEventRecord(s->ev[2], st);
    {
        NvtxRange nv("tt_execute_sharded unpack");
        if (launch_plan(*s->unpack, s->recv, out_local, p->stream) != 0) return TT_CUDA_ERROR;
    }
    cudaEventRecord(s->ev[3], st);
    s->timed = true;
    return TT_SUCCESS;
}

tt_status_t tt_sharded_timings(tt_plan_t plan, float* ms3) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    if (ms3 == nullptr) return TT_INVALID_PARAMETER;
    ShardInfo* s = p->shard;
    ms3[0] = ms3[1] = ms3[2] = 0.f;
    if (!s->redistribute || !s->timed) return TT_SUCCESS;
    if (cudaEventSynchronize(s->ev[3]) != cudaSuccess) { cudaGetLastError(); return TT_CUDA_ERROR; }
    if (s->chunks > 1) {  // spans: packs on the plan stream, all-to-alls, unpacks (they overlap)
        if (cudaEventElapsedTime(&ms3[0], s->ev[0], s->ev[1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms3[1], s->evT[0], s->evT[1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms3[2], s->evT[2], s->evT[3]) != cudaSuccess) {
            cudaGetLastError();
            return TT_CUDA_ERROR;
        }
        return TT_SUCCESS;
    }
    for (int i = 0; i < 3; ++i)
        if (cudaEventElapsedTime(&ms3[i], s->ev[i], s->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            return TT_CUDA_ERROR;
        }
    if (s->p2p && s->sig) {  // a peer that never reached a barrier
        int err = 0;
        if (cudaMemcpy(&err, s->sig + s->nranks, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return TT_CUDA_ERROR;
        }
        if (err != 0) return TT_CUDA_ERROR;
    }
    return TT_SUCCESS;
}

tt_status_t tt_plan_shard_dims(tt_plan_t plan, int64_t* local_in_dims, int64_t* local_out_dims) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    for (size_t i = 0; i < s->local_in.size(); ++i) {
        if (local_in_dims) local_in_dims[i] = s->local_in[i];
        if (local_out_dims) local_out_dims[i] = s->local_out[i];
    }
    return TT_SUCCESS;
}

tt_status_t tt_plan_sharded_p2p(tt_plan_t* plan, tt_comm_t comm, int nranks, int proc, int ndims,
                                const int64_t* global_dims, const int* perm, size_t elem_size,
                                tt_stream_t stream) {
    return tt_plan_sharded_p2p_ex(plan, comm, nranks, proc, ndims, global_dims, perm, elem_size, stream,
                                  nullptr);
}

tt_status_t tt_plan_sharded_p2p_ex(tt_plan_t* plan, tt_comm_t comm, int nranks, int proc, int ndims,
                                   const int64_t* global_dims, const int* perm, size_t elem_size,
                                   tt_stream_t stream, const tt_plan_options_t* opts) {
    if (plan == nullptr || ndims < 1) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    tt_comm_impl* c = nullptr;
    if (comm != nullptr) {
        c = as_comm(comm);
        if (c == nullptr || c->nranks != nranks || c->rank != proc) return TT_INVALID_PARAMETER;
    }
    if (nranks < 1 || nranks > kMaxPeers) return TT_UNSUPPORTED;
    DeviceInfo dev;
    tt_status_t st = query_device(dev);
    if (st != TT_SUCCESS) return st;
    if (c && dev.device != c->device) return TT_INVALID_DEVICE;
    Plan* p = nullptr;
    st = build_shard_n(&p, c, nranks, proc, ndims, global_dims, perm, elem_size, stream, dev,
                       &cuda_occupancy, true, opts && opts->force_redistribute);
    if (st != TT_SUCCESS) return st;
    ShardInfo* s = p->shard;
    for (auto& e : s->ev) {
        if (cudaEventCreate(&e) != cudaSuccess) {
            cudaGetLastError();
            destroy_plan(p);
            return TT_CUDA_ERROR;
        }
    }
    *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return TT_SUCCESS;
}

tt_status_t tt_plan_sharded_p2p_offline(tt_plan_t* plan, int nranks, int proc, int ndims,
                                        const int64_t* global_dims, const int* perm,
                                        size_t elem_size) {
    if (plan == nullptr || ndims < 1) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    if (nranks < 1 || nranks > kMaxPeers) return TT_UNSUPPORTED;
    DeviceInfo dev;
    dev.device = -1;
    Plan* p = nullptr;
    tt_status_t st = build_shard_n(&p, nullptr, nranks, proc, ndims, global_dims, perm, elem_size,
                                   nullptr, dev, nullptr, true);
    if (st == TT_SUCCESS) *plan = reinterpret_cast<tt_plan_t>(publish_handle(p));
    return st;
}

tt_status_t tt_sharded_register_output(tt_plan_t plan, void* out_local) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    if (!s->p2p || s->comm == nullptr) return TT_INVALID_PLAN;
    if (out_local == nullptr || (reinterpret_cast<uintptr_t>(out_local) & (uintptr_t)(s->esize - 1)))
        return TT_INVALID_PARAMETER;
    if (s->reg_out != nullptr) return TT_INVALID_PARAMETER;  // once per plan
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    const int P = s->nranks;
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    RegRecord mine;
    const tt_status_t local = make_record(s, d, out_local, mine);
    // all-gather the records with the communicator (no host-side rendezvous);
    // a rank that failed above still joins with ok = 0 so no peer blocks
    void* dbuf = nullptr;
    std::vector<RegRecord> all(P);
    if (cudaMalloc(&dbuf, (size_t)(P + 1) * sizeof(RegRecord)) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    char* dsend = static_cast<char*>(dbuf) + (size_t)P * sizeof(RegRecord);
    tt_status_t rc = TT_SUCCESS;
    if (cudaMemcpyAsync(dsend, &mine, sizeof(mine), cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = TT_CUDA_ERROR;
    else if (ncclAllGather(dsend, dbuf, sizeof(RegRecord), ncclUint8, s->comm->nccl, st) != ncclSuccess)
        rc = TT_NCCL_ERROR;
    else if (cudaMemcpyAsync(all.data(), dbuf, (size_t)P * sizeof(RegRecord), cudaMemcpyDeviceToHost,
                             st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        rc = TT_CUDA_ERROR;
    cudaFree(dbuf);
    if (rc != TT_SUCCESS) { cudaGetLastError(); return rc; }
    if (local != TT_SUCCESS) return local;
    return open_records(s, out_local, all.data());
}

tt_status_t tt_sharded_export_record(tt_plan_t plan, void* out_local, void* record) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    if (!s->p2p) return TT_INVALID_PLAN;
    if (record == nullptr || out_local == nullptr ||
        (reinterpret_cast<uintptr_t>(out_local) & (uintptr_t)(s->esize - 1)))
        return TT_INVALID_PARAMETER;
    if (s->reg_out != nullptr) return TT_INVALID_PARAMETER;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    RegRecord mine;
    const tt_status_t st = make_record(s, d, out_local, mine);
    std::memcpy(record, &mine, sizeof(mine));   // ok = 0 on failure: peers see it
    if (st == TT_SUCCESS) s->exported = out_local;
    return st;
}

tt_status_t tt_sharded_import_records(tt_plan_t plan, const void* records) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    if (!s->p2p) return TT_INVALID_PLAN;
    if (records == nullptr || s->exported == nullptr) return TT_INVALID_PARAMETER;
    if (s->reg_out != nullptr) return TT_INVALID_PARAMETER;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    std::vector<RegRecord> all(s->nranks);
    std::memcpy(all.data(), records, all.size() * sizeof(RegRecord));
    return open_records(s, s->exported, all.data());
}

tt_status_t tt_execute_sharded_p2p(tt_plan_t plan, const void* in_local, void* const* out_slabs) {
    Plan* p = as_plan(plan);
    if (p == nullptr || p->shard == nullptr) return TT_INVALID_PLAN;
    ShardInfo* s = p->shard;
    if (in_local == nullptr || out_slabs == nullptr) return TT_INVALID_PARAMETER;
    uintptr_t bits = reinterpret_cast<uintptr_t>(in_local);
    for (int q = 0; q < s->nranks; ++q) {
        if (out_slabs[q] == nullptr || out_slabs[q] == in_local) return TT_INVALID_PARAMETER;
        bits |= reinterpret_cast<uintptr_t>(out_slabs[q]);
    }
    if ((bits & (uintptr_t)(s->esize - 1)) != 0) return TT_INVALID_PARAMETER;
    if (p->device < 0) return TT_INVALID_DEVICE;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    if (!s->redistribute)
        return launch_plan(*s->local, in_local, out_slabs[s->proc], p->stream) == 0 ? TT_SUCCESS
                                                                                   : TT_CUDA_ERROR;
    if (!s->p2p) return TT_INVALID_PLAN;
    return launch_fused(s, in_local, out_slabs, p->stream);
}

}  // extern "C\"
