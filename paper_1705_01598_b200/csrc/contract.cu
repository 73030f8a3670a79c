// contract.cu -- TTGT tensor contraction (SURVEY f-4): the workload of the
// paper's Section 3.4, D = alpha * L . R + beta * D, computed as
// Transpose-Transpose-GEMM-Transpose: "a binary tensor contraction can
// involve up to four tensor transposes (two forward transposes for the two
// input tensors, one forward and one backward transpose for the output
// tensor)".  The transposes are this library's plans; the GEMM is a
// plain cuBLAS GEMM (a library GEMM, not the product).
//
//   modes: integer labels, one per dimension (dim 0 = stride-1, as tt_plan).
//   M = free labels of L in D's order, N = free labels of R in D's order,
//   K = contracted labels (in L and R, not in D) in L's order.
//   L -> L' = [M.., K..] (m x k, column-major)   or used as is: [K.., M..] = op T
//   R -> R' = [K.., N..] (k x n)                 or used as is: [N.., K..] = op T
//   D  = [M.., N..] : GEMM writes D directly (alpha, beta in the GEMM)
//   D  = [N.., M..] : GEMM of the transposed problem writes D directly
//   else            : GEMM into workspace W = [M.., N..], then W -> D by a
//                     permutation plan (plain when beta == 0, the accumulate
//                     form of tt_execute_scaled otherwise).
//
// Forward transposes are skipped when the labels are already in GEMM order
// (identity permutation), so a contraction runs 1 to 4 launches besides the
// GEMM.  Time is measured from the first transpose to the end of the last
// operation by the caller with CUDA events on the plan's stream;
// tt_contract_timings splits it by step.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "tt_internal.h"

namespace tt {

struct Operand {
    Plan* plan = nullptr;        // forward transpose (null: used as stored)
    void* buf = nullptr;         // workspace of the transposed operand
    bool trans = false;          // GEMM op: T (stored as [K.., M..] / [N.., K..])
    std::vector<int> perm;       // transpose permutation (described)
};

struct Contract {
    int device = -1;
    void* stream = nullptr;
    int esize = 8;
    cublasHandle_t blas = nullptr;
    int64_t m = 1, n = 1, k = 1;
    int64_t volL = 1, volR = 1, volD = 1;
    std::vector<int> modesL, modesR, modesD;
    std::vector<int64_t> dimsL, dimsR, dimsD;
    Operand L, R;
    bool swapMN = false;           // GEMM computes D = (L'R')^T directly ([N.., M..] order)
    bool direct = true;            // GEMM writes D (else W + back transpose)
    Plan* back = nullptr;          // W -> D, beta == 0
    Plan* backAcc = nullptr;       // W -> D, accumulate form (beta != 0); null if unsupported
    void* W = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool timed = false;
};

static void destroy_contract(Contract* c) {
    if (!c) return;
    destroy_plan(c->L.plan);
    destroy_plan(c->R.plan);
    destroy_plan(c->back);
    destroy_plan(c->backAcc);
    if (c->L.buf) cudaFree(c->L.buf);
    if (c->R.buf) cudaFree(c->R.buf);
    if (c->W) cudaFree(c->W);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->blas) cublasDestroy(c->blas);
    delete c;
}

static int find(const std::vector<int>& v, int x) {
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i] == x) return (int)i;
    return -1;
}

static bool is_identity(const std::vector<int>& p) {
    for (size_t i = 0; i < p.size(); ++i)
        if (p[i] != (int)i) return false;
    return true;
}

// Build the forward transpose of one operand to the label order `want`
// (a permutation of its labels): identity -> as stored; `alt` order
// identity -> as stored with GEMM op T; else a permutation plan + workspace.
static tt_status_t build_operand(Operand& op, const std::vector<int>& modes,
                                 const std::vector<int64_t>& dims, const std::vector<int>& want,
                                 const std::vector<int>& alt, int64_t vol, size_t esize,
                                 void* stream, const DeviceInfo& dev, bool alloc) {
    std::vector<int> p(want.size()), pa(alt.size());
    for (size_t j = 0; j < want.size(); ++j) p[j] = find(modes, want[j]);
    for (size_t j = 0; j < alt.size(); ++j) pa[j] = find(modes, alt[j]);
    if (is_identity(p)) return TT_SUCCESS;
    if (is_identity(pa)) { op.trans = true; return TT_SUCCESS; }
    op.perm = p;
    tt_status_t st = create_plan(&op.plan, (int)modes.size(), dims.data(), p.data(), esize, stream,
                                 dev, nullptr, alloc ? &cuda_occupancy : nullptr);
    if (st != TT_SUCCESS) return st;
    if (alloc && cudaMalloc(&op.buf, (size_t)vol * esize) != cudaSuccess) {
        cudaGetLastError();
        return TT_CUDA_ERROR;
    }
    return TT_SUCCESS;
}

static tt_status_t build_contract(Contract** out, int rD, const int* mD, int rL, const int64_t* dL,
                                  const int* mL, int rR, const int64_t* dR, const int* mR,
                                  size_t esize, void* stream, bool online) {
    *out = nullptr;
    if (rD < 0 || rL < 0 || rR < 0 || rD > TT_MAX_RANK || rL > TT_MAX_RANK || rR > TT_MAX_RANK)
        return TT_INVALID_PARAMETER;
    if ((rD && !mD) || (rL && (!dL || !mL)) || (rR && (!dR || !mR))) return TT_INVALID_PARAMETER;
    if (esize != 4 && esize != 8) return TT_UNSUPPORTED;
    Contract* c = new (std::nothrow) Contract();
    if (!c) return TT_INTERNAL_ERROR;
    c->esize = (int)esize;
    c->stream = stream;
    c->modesL.assign(mL, mL + rL);
    c->modesR.assign(mR, mR + rR);
    c->modesD.assign(mD, mD + rD);
    c->dimsL.assign(dL, dL + rL);
    c->dimsR.assign(dR, dR + rR);
    auto fail = [&](tt_status_t s) { destroy_contract(c); return s; };
    // labels: distinct within a tensor, non-negative, extents >= 1
    auto distinct = [](const std::vector<int>& v) {
        for (size_t i = 0; i < v.size(); ++i) {
            if (v[i] < 0) return false;
            for (size_t j = 0; j < i; ++j)
                if (v[i] == v[j]) return false;
        }
        return true;
    };
    if (!distinct(c->modesL) || !distinct(c->modesR) || !distinct(c->modesD))
        return fail(TT_INVALID_PARAMETER);
    for (int64_t x : c->dimsL) if (x < 1) return fail(TT_INVALID_PARAMETER);
    for (int64_t x : c->dimsR) if (x < 1) return fail(TT_INVALID_PARAMETER);
    std::vector<int> M, N, K;
    for (int l : c->modesD) {
        const int a = find(c->modesL, l), b = find(c->modesR, l);
        if (a >= 0 && b >= 0) return fail(TT_UNSUPPORTED);       // batch (Hadamard) label
        if (a < 0 && b < 0) return fail(TT_INVALID_PARAMETER);   // D label from nowhere
        if (a >= 0) { M.push_back(l); c->dimsD.push_back(c->dimsL[a]); }
        else { N.push_back(l); c->dimsD.push_back(c->dimsR[b]); }
    }
    for (size_t i = 0; i < c->modesL.size(); ++i) {
        const int l = c->modesL[i];
        if (find(c->modesD, l) >= 0) continue;
        const int b = find(c->modesR, l);
        if (b < 0) return fail(TT_INVALID_PARAMETER);            // summed over one tensor only
        if (c->dimsR[b] != c->dimsL[i]) return fail(TT_INVALID_PARAMETER);
        K.push_back(l);
    }
    for (int l : c->modesR)
        if (find(c->modesD, l) < 0 && find(c->modesL, l) < 0) return fail(TT_INVALID_PARAMETER);
    long double vl = 1, vr = 1, vd = 1;
    for (int64_t x : c->dimsL) vl *= x;
    for (int64_t x : c->dimsR) vr *= x;
    for (int64_t x : c->dimsD) vd *= x;
    if (vl * esize >= (long double)(1LL << 62) || vr * esize >= (long double)(1LL << 62) ||
        vd * esize >= (long double)(1LL << 62))
        return fail(TT_INVALID_PARAMETER);
    c->volL = (int64_t)vl;
    c->volR = (int64_t)vr;
    c->volD = (int64_t)vd;
    for (int l : M) c->m *= c->dimsL[find(c->modesL, l)];
    for (int l : N) c->n *= c->dimsR[find(c->modesR, l)];
    for (int l : K) c->k *= c->dimsL[find(c->modesL, l)];
    // cuBLAS takes int dimensions
    if (c->m >= (1LL << 31) || c->n >= (1LL << 31) || c->k >= (1LL << 31)) return fail(TT_UNSUPPORTED);

    DeviceInfo dev;
    if (online) {
        tt_status_t st = query_device(dev);
        if (st != TT_SUCCESS) return fail(st);
    } else {
        dev.device = -1;
    }
    c->device = dev.device;
    std::vector<int> MK = M, KM = K, KN = K, NK = N;
    MK.insert(MK.end(), K.begin(), K.end());
    KM.insert(KM.end(), M.begin(), M.end());
    KN.insert(KN.end(), N.begin(), N.end());
    NK.insert(NK.end(), K.begin(), K.end());
    tt_status_t st = build_operand(c->L, c->modesL, c->dimsL, MK, KM, c->volL, esize, stream, dev, online);
    if (st != TT_SUCCESS) return fail(st);
    st = build_operand(c->R, c->modesR, c->dimsR, KN, NK, c->volR, esize, stream, dev, online);
    if (st != TT_SUCCESS) return fail(st);
    // output: [M.., N..] or [N.., M..] in D's order -> GEMM writes D
    std::vector<int> MN = M, NM = N;
    MN.insert(MN.end(), N.begin(), N.end());
    NM.insert(NM.end(), M.begin(), M.end());
    if (MN == c->modesD) {
        c->direct = true;
    } else if (NM == c->modesD) {
        c->direct = true;
        c->swapMN = true;
    } else {
        c->direct = false;
        // W = [M.., N..] with extents; back permutation W -> D
        std::vector<int64_t> wd;
        for (int l : MN) wd.push_back(c->dimsD[find(c->modesD, l)]);
        std::vector<int> bp(rD);
        for (int j = 0; j < rD; ++j) bp[j] = find(MN, c->modesD[j]);
        st = create_plan(&c->back, rD, wd.data(), bp.data(), esize, stream, dev, nullptr,
                         online ? &cuda_occupancy : nullptr);
        if (st != TT_SUCCESS) return fail(st);
        tt_plan_options_t o;
        std::memset(&o, 0, sizeof(o));
        o.accumulate = 1;
        if (create_plan(&c->backAcc, rD, wd.data(), bp.data(), esize, stream, dev, &o,
                        online ? &cuda_occupancy : nullptr) != TT_SUCCESS)
            c->backAcc = nullptr;  // beta != 0 then unsupported (64-bit indices)
        if (online && cudaMalloc(&c->W, (size_t)c->volD * esize) != cudaSuccess) {
            cudaGetLastError();
            return fail(TT_CUDA_ERROR);
        }
    }
    if (online) {
        if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS ||
            cublasSetStream(c->blas, static_cast<cudaStream_t>(stream)) != CUBLAS_STATUS_SUCCESS ||
            cublasSetPointerMode(c->blas, CUBLAS_POINTER_MODE_HOST) != CUBLAS_STATUS_SUCCESS ||
            cublasSetMathMode(c->blas, CUBLAS_DEFAULT_MATH) != CUBLAS_STATUS_SUCCESS)
            return fail(TT_CUDA_ERROR);
        for (auto& e : c->ev)
            if (cudaEventCreate(&e) != cudaSuccess) {
                cudaGetLastError();
                return fail(TT_CUDA_ERROR);
            }
    }
    *out = c;
    return TT_SUCCESS;
}

static std::string describe_contract(const Contract& c) {
    std::ostringstream o;
    auto arr = [&](const auto& v) {
        o << "[";
        for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << (long long)v[i];
        o << "]";
    };
    o << "{\"version\":" << TT_VERSION << ",\"contraction\":true,\"elem_size\":" << c.esize
      << ",\"m\":" << c.m << ",\"n\":" << c.n << ",\"k\":" << c.k << ",\"dims_d\":";
    arr(c.dimsD);
    o << ",\"transpose_l\":" << (c.L.plan ? "true" : "false") << ",\"op_l\":\"" << (c.L.trans ? "T" : "N")
      << "\",\"transpose_r\":" << (c.R.plan ? "true" : "false") << ",\"op_r\":\"" << (c.R.trans ? "T" : "N")
      << "\",\"swap_mn\":" << (c.swapMN ? "true" : "false")
      << ",\"transpose_d\":" << (c.direct ? "false" : "true");
    if (c.L.plan) { o << ",\"perm_l\":"; arr(c.L.perm); o << ",\"plan_l\":" << describe_json(*c.L.plan); }
    if (c.R.plan) { o << ",\"perm_r\":"; arr(c.R.perm); o << ",\"plan_r\":" << describe_json(*c.R.plan); }
    if (c.back) o << ",\"plan_d\":" << describe_json(*c.back);
    o << ",\"launches\":"
      << (c.L.plan ? 1 : 0) + (c.R.plan ? 1 : 0) + (c.direct ? 0 : 1) << "}";
    return o.str();
}

}  // namespace tt

using namespace tt;

static Contract* as_contract(tt_contract_t h) {
    return handle_live(h) ? reinterpret_cast<Contract*>(h) : nullptr;
}

extern "C" {

tt_status_t tt_contract_plan(tt_contract_t* plan, int rank_d, const int* modes_d, int rank_l,
                             const int64_t* dims_l, const int* modes_l, int rank_r,
                             const int64_t* dims_r, const int* modes_r, size_t elem_size,
                             tt_stream_t stream) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    Contract* c = nullptr;
    tt_status_t st = build_contract(&c, rank_d, modes_d, rank_l, dims_l, modes_l, rank_r, dims_r,
                                    modes_r, elem_size, stream, true);
    if (st == TT_SUCCESS) *plan = reinterpret_cast<tt_contract_t>(publish_handle(c));
    return st;
}

tt_status_t tt_contract_plan_offline(tt_contract_t* plan, int rank_d, const int* modes_d, int rank_l,
                                     const int64_t* dims_l, const int* modes_l, int rank_r,
                                     const int64_t* dims_r, const int* modes_r, size_t elem_size) {
    if (plan == nullptr) return TT_INVALID_PARAMETER;
    *plan = nullptr;
    Contract* c = nullptr;
    tt_status_t st = build_contract(&c, rank_d, modes_d, rank_l, dims_l, modes_l, rank_r, dims_r,
                                    modes_r, elem_size, nullptr, false);
    if (st == TT_SUCCESS) *plan = reinterpret_cast<tt_contract_t>(publish_handle(c));
    return st;
}

tt_status_t tt_contract_execute(tt_contract_t plan, const void* l, const void* r, void* d,
                                double alpha, double beta) {
    Contract* c = as_contract(plan);
    if (c == nullptr) return TT_INVALID_PLAN;
    if (!l || !r || !d || d == l || d == r) return TT_INVALID_PARAMETER;
    if (((reinterpret_cast<uintptr_t>(l) | reinterpret_cast<uintptr_t>(r) |
          reinterpret_cast<uintptr_t>(d)) & (uintptr_t)(c->esize - 1)) != 0)
        return TT_INVALID_PARAMETER;
    if (c->device < 0) return TT_INVALID_DEVICE;
    int dv = -1;
    if (cudaGetDevice(&dv) != cudaSuccess || dv != c->device) { cudaGetLastError(); return TT_INVALID_DEVICE; }
    if (!c->direct && beta != 0.0 && c->backAcc == nullptr) return TT_UNSUPPORTED;
    cudaStream_t s = static_cast<cudaStream_t>(c->stream);
    cudaEventRecord(c->ev[0], s);
    const void* Lp = l;
    if (c->L.plan) {
        if (launch_plan(*c->L.plan, l, c->L.buf, c->stream) != 0) return TT_CUDA_ERROR;
        Lp = c->L.buf;
    }
    cudaEventRecord(c->ev[1], s);
    const void* Rp = r;
    if (c->R.plan) {
        if (launch_plan(*c->R.plan, r, c->R.buf, c->stream) != 0) return TT_CUDA_ERROR;
        Rp = c->R.buf;
    }
    cudaEventRecord(c->ev[2], s);
    // column-major GEMM: X (m x n) = op(L') (m x k) . op(R') (k x n)
    const int m = (int)c->m, n = (int)c->n, k = (int)c->k;
    const cublasOperation_t oL = c->L.trans ? CUBLAS_OP_T : CUBLAS_OP_N;
    const cublasOperation_t oR = c->R.trans ? CUBLAS_OP_T : CUBLAS_OP_N;
    const int ldL = c->L.trans ? k : m;   // stored [K.., M..] is k x m
    const int ldR = c->R.trans ? n : k;   // stored [N.., K..] is n x k
    void* X = c->direct ? d : c->W;
    const double bX = c->direct ? beta : 0.0;
    cublasStatus_t bs;
    if (!c->swapMN) {
        if (c->esize == 8) {
            bs = cublasDgemm(c->blas, oL, oR, m, n, k, &alpha, (const double*)Lp, ldL, (const double*)Rp,
                             ldR, &bX, (double*)X, m);
        } else {
            const float a = (float)alpha, b = (float)bX;
            bs = cublasSgemm(c->blas, oL, oR, m, n, k, &a, (const float*)Lp, ldL, (const float*)Rp, ldR,
                             &b, (float*)X, m);
        }
    } else {
        // D = X^T (n x m) = op(R')^T . op(L')^T
        const cublasOperation_t tR = oR == CUBLAS_OP_N ? CUBLAS_OP_T : CUBLAS_OP_N;
        const cublasOperation_t tL = oL == CUBLAS_OP_N ? CUBLAS_OP_T : CUBLAS_OP_N;
        if (c->esize == 8) {
            bs = cublasDgemm(c->blas, tR, tL, n, m, k, &alpha, (const double*)Rp, ldR, (const double*)Lp,
                             ldL, &bX, (double*)X, n);
        } else {
            const float a = (float)alpha, b = (float)bX;
            bs = cublasSgemm(c->blas, tR, tL, n, m, k, &a, (const float*)Rp, ldR, (const float*)Lp, ldL,
                             &b, (float*)X, n);
        }
    }
    if (bs != CUBLAS_STATUS_SUCCESS) return TT_CUDA_ERROR;
    cudaEventRecord(c->ev[3], s);
    if (!c->direct) {
        int e = beta == 0.0 ? launch_plan(*c->back, c->W, d, c->stream)
                            : launch_plan_scaled(*c->backAcc, c->W, d, c->stream, 1.0, beta);
        if (e != 0) return TT_CUDA_ERROR;
    }
    cudaEventRecord(c->ev[4], s);
    c->timed = true;
    return TT_SUCCESS;
}

tt_status_t tt_contract_timings(tt_contract_t plan, float* ms4) {
    Contract* c = as_contract(plan);
    if (c == nullptr) return TT_INVALID_PLAN;
    if (ms4 == nullptr) return TT_INVALID_PARAMETER;
    for (int i = 0; i < 4; ++i) ms4[i] = 0.f;
    if (!c->timed) return TT_SUCCESS;
    if (cudaEventSynchronize(c->ev[4]) != cudaSuccess) { cudaGetLastError(); return TT_CUDA_ERROR; }
    for (int i = 0; i < 4; ++i)
        if (cudaEventElapsedTime(&ms4[i], c->ev[i], c->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            return TT_CUDA_ERROR;
        }
    return TT_SUCCESS;
}

tt_status_t tt_contract_describe(tt_contract_t plan, char* buf, size_t len) {
    Contract* c = as_contract(plan);
    if (c == nullptr) return TT_INVALID_PLAN;
    if (buf == nullptr || len == 0) return TT_INVALID_PARAMETER;
    const std::string s = describe_contract(*c);
    std::strncpy(buf, s.c_str(), len - 1);
    buf[len - 1] = 0;
    return s.size() + 1 > len ? TT_BUFFER_TOO_SMALL : TT_SUCCESS;
}

tt_status_t tt_contract_destroy(tt_contract_t plan) {
    if (!retire_handle(plan)) return TT_INVALID_PLAN;  // NULL or already destroyed
    destroy_contract(reinterpret_cast<Contract*>(plan));
    return TT_SUCCESS;
}

}  // extern "C"
