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
// Both local steps are ordinary single-GPU plans (planner.cpp + kernels.cu).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "tt_internal.h"

namespace tt {

struct tt_comm_impl {
    uint32_t magic = 0x5454434du;  // "TTCM"
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
};

void destroy_shard(ShardInfo* s) {
    if (!s) return;
    destroy_plan(s->local);
    destroy_plan(s->pack);
    destroy_plan(s->unpack);
    if (s->send) cudaFree(s->send);
    if (s->recv) cudaFree(s->recv);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    delete s;
}

int shard_launches(const ShardInfo* s) {
    if (!s->redistribute) return 1;
    return s->nranks > 1 ? 3 : 2;  // pack, (NCCL all-to-all), unpack
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
      << ",\"rank\":" << s->rank << ",\"mode\":\"" << (s->redistribute ? "redistribute" : "local")
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
    if (s->pack) o << ",\"pack\":" << describe_json(*s->pack);
    if (s->unpack) o << ",\"unpack\":" << describe_json(*s->unpack);
    o << "}";
    return o.str();
}

// Geometry + sub-plans; comm may be null (offline).
static tt_status_t build_shard_n(Plan** out, tt_comm_impl* comm, int nranks, int rank, int n,
                                 const int64_t* gd, const int* perm, size_t esize, void* stream,
                                 const DeviceInfo& dev, OccupancyFn occ) {
    *out = nullptr;
    tt_status_t st = validate(n, gd, perm, esize);
    if (st != TT_SUCCESS) return st;
    if (nranks < 1 || rank < 0 || rank >= nranks) return TT_INVALID_PARAMETER;
    const int P = nranks;
    const int t = perm[n - 1];
    if (gd[n - 1] % P != 0) return TT_UNSUPPORTED;
    // TT_SHARD_FORCE_REDIST=1 (tests): take the pack / all-to-all / unpack path
    // even with one rank, so the NCCL path runs on a single-GPU box
    const char* force = std::getenv("TT_SHARD_FORCE_REDIST");
    const bool redist = (t != n - 1) && (P > 1 || (force && force[0] == '1'));
    if (redist && gd[t] % P != 0) return TT_UNSUPPORTED;

    ShardInfo* s = new (std::nothrow) ShardInfo();
    Plan* outer = new (std::nothrow) Plan();
    if (!s || !outer) { delete s; delete outer; return TT_INTERNAL_ERROR; }
    s->comm = comm;
    s->nranks = P;
    s->rank = rank;
    s->esize = (int)esize;
    s->redistribute = redist;
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

    // pack: split input dim t into (c = D[t]/P, P), P-part outermost
    const int64_t c = gd[t] / P;
    std::vector<int64_t> pd;
    auto ni = [&](int i) { return i < t ? i : (i == t ? t : i + 1); };
    for (int i = 0; i < n; ++i) {
        if (i == t) { pd.push_back(c); pd.push_back(P); }
        else pd.push_back(L[i]);
    }
    std::vector<int> pp;
    for (int j = 0; j < n; ++j) pp.push_back(ni(perm[j]));
    pp.push_back(t + 1);
    st = create_plan(&s->pack, n + 1, pd.data(), pp.data(), esize, stream, dev, nullptr, occ);
    if (st != TT_SUCCESS) { destroy_plan(outer); return st; }

    // unpack: received [e'_0 .. e'_{n-1}, P_src] -> move P_src after j*
    std::vector<int64_t> ep(n);
    int jstar = -1;
    for (int j = 0; j < n; ++j) {
        ep[j] = (j == n - 1) ? c : L[perm[j]];
        if (perm[j] == n - 1) jstar = j;
    }
    int64_t inner = 1, middle = 1;
    for (int j = 0; j <= jstar; ++j) inner *= ep[j];
    for (int j = jstar + 1; j < n; ++j) middle *= ep[j];
    const int64_t ud[3] = {inner, middle, (int64_t)P};
    const int up[3] = {0, 2, 1};
    st = create_plan(&s->unpack, 3, ud, up, esize, stream, dev, nullptr, occ);
    if (st != TT_SUCCESS) { destroy_plan(outer); return st; }
    s->a2a_count = (size_t)(shard_vol / P);
    *out = outer;
    return TT_SUCCESS;
}

}  // namespace tt

using namespace tt;

static tt_comm_impl* as_comm(tt_comm_t c) {
    tt_comm_impl* p = reinterpret_cast<tt_comm_impl*>(c);
    if (p == nullptr || p->magic != 0x5454434du) return nullptr;
    return p;
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
    *comm = reinterpret_cast<tt_comm_t>(c);
    return TT_SUCCESS;
}

tt_status_t tt_comm_destroy(tt_comm_t comm) {
    tt_comm_impl* c = as_comm(comm);
    if (c == nullptr) return TT_INVALID_PARAMETER;
    ncclResult_t r = ncclCommDestroy(c->nccl);
    c->magic = 0;
    delete c;
    return r == ncclSuccess ? TT_SUCCESS : TT_NCCL_ERROR;
}

tt_status_t tt_plan_sharded(tt_plan_t* plan, tt_comm_t comm, int ndims, const int64_t* global_dims,
                            const int* perm, size_t elem_size, tt_stream_t stream) {
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
                       &cuda_occupancy);
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
    for (auto& e : s->ev) {
        if (cudaEventCreate(&e) != cudaSuccess) {
            cudaGetLastError();
            destroy_plan(p);
            return TT_CUDA_ERROR;
        }
    }
    *plan = reinterpret_cast<tt_plan_t>(p);
    return TT_SUCCESS;
}

tt_status_t tt_plan_sharded_offline(tt_plan_t* plan, int nranks, int rank, int ndims,
                                    const int64_t* global_dims, const int* perm, size_t elem_size) {
    if (ndims < 1) return TT_INVALID_PARAMETER;
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    DeviceInfo dev;
    dev.device = -1;
    Plan* p = nullptr;
    tt_status_t st = build_shard_n(&p, nullptr, nranks, rank, ndims, global_dims, perm, elem_size,
                                   nullptr, dev, nullptr);
    if (st == TT_SUCCESS) *plan = reinterpret_cast<tt_plan_t>(p);
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
    if (s->comm == nullptr || p->device < 0) return TT_INVALID_DEVICE;
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != p->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    cudaStream_t st = static_cast<cudaStream_t>(p->stream);
    if (!s->redistribute)
        return launch_plan(*s->local, in_local, out_local, p->stream) == 0 ? TT_SUCCESS : TT_CUDA_ERROR;
    cudaEventRecord(s->ev[0], st);
    if (launch_plan(*s->pack, in_local, s->send, p->stream) != 0) return TT_CUDA_ERROR;
    cudaEventRecord(s->ev[1], st);
    const ncclDataType_t dt = s->esize == 4 ? ncclUint32 : ncclUint64;
    if (ncclAlltoAll(s->send, s->recv, s->a2a_count, dt, s->comm->nccl, st) != ncclSuccess)
        return TT_NCCL_ERROR;
    cudaEventRecord(s->ev[2], st);
    if (launch_plan(*s->unpack, s->recv, out_local, p->stream) != 0) return TT_CUDA_ERROR;
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
    for (int i = 0; i < 3; ++i)
        if (cudaEventElapsedTime(&ms3[i], s->ev[i], s->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            return TT_CUDA_ERROR;
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

}  // extern "C"
