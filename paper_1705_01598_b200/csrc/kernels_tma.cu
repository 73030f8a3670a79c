// kernels_tma.cu -- 2-D tiled transpose (Tiled class) staged by
// the Tensor Memory Accelerator.
//
// Citations: P:Lnn = PAPER.md line nn (arXiv 1705.01598).
//
// A fused problem of the Tiled class has input dim A = 0 (stride 1) and the
// output-fastest input dim B = perm[0]; the other dims are batch dims.  When
// every stride is a multiple of 16 bytes (cuTensorMapEncodeTiled's rule:
// d_A * E and d_B * E multiples of 16), the input is a TMA tensor of rank
// 2 + batch (<= 5) and the output another one with A and B swapped.  Per tile:
//   * one elected thread loads the TA x TB input box with
//     cp.async.bulk.tensor (UTMALDG) into a ring of S stages, completing on
//     the stage's mbarrier (expect_tx = box bytes); boxes crossing the tensor
//     ends are zero-filled by the hardware (ragged tiles need no masks);
//   * all threads transpose the box in shared memory into an output box
//     along a diagonal (lane l takes a = a0 + l, b = (bb + l) mod TB), which
//     is bank-conflict free both ways without padding -- TMA boxes are dense
//     (the L x (L+1) padding of P:L123 is not available);
//   * the elected thread stores the output box with a TMA tensor store
//     (UTMASTG), which clips at the tensor ends; two output boxes alternate.
// Global traffic never goes through registers or the LSU; the only per-element
// thread work is one LDS and one STS.
#include <cuda.h>

#include "kern_common.cuh"
#include "kern_pick.h"

namespace tt {

__device__ __forceinline__ void mbar_init_t(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_t(uint32_t a, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

template <int R>
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* map, const int* c, uint32_t mbar) {
    if constexpr (R == 2)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"(map), "r"(c[0]), "r"(c[1]), "r"(mbar) : "memory");
    else if constexpr (R == 3)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(dst), "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(mbar) : "memory");
    else if constexpr (R == 4)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(dst), "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(mbar) : "memory");
    else
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(dst), "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(mbar) : "memory");
}

template <int R>
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const int* c, uint32_t src) {
    if constexpr (R == 2)
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(map), "r"(c[0]), "r"(c[1]), "r"(src) : "memory");
    else if constexpr (R == 3)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                     ::"l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(src) : "memory");
    else if constexpr (R == 4)
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                     ::"l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(src) : "memory");
    else
        asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                     ::"l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(src) : "memory");
}

// Tile t -> box coordinates: B-chunks fastest, then A-chunks, then the batch
// dims (the 2-D kernels' default order); in = (a0, b0, batch...), out =
// (b0, a0, batch...).
__device__ __forceinline__ void tma_coords(const Tma2DParams& p, uint32_t t, int* ci, int* co) {
    const uint32_t cb = t % (uint32_t)p.nB;
    uint32_t r = t / (uint32_t)p.nB;
    const uint32_t ca = r % (uint32_t)p.nA;
    r /= (uint32_t)p.nA;
    ci[0] = (int)(ca * p.TA);
    ci[1] = (int)(cb * p.TB);
    co[0] = ci[1];
    co[1] = ci[0];
    for (int k = 0; k < 3; ++k) {
        int x = 0;
        if (k < p.nb) {
            x = (int)(r % (uint32_t)p.bExt[k]);
            r /= (uint32_t)p.bExt[k];
        }
        ci[2 + k] = x;
        co[2 + k] = x;
    }
}

template <typename W, int TA, int TB, int S, int R>
__global__ void __launch_bounds__(256) tiled2d_tma_kernel(const __grid_constant__ Tma2DParams p) {
    constexpr uint32_t BOX = TA * TB * sizeof(W);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // 128-byte aligned base for the boxes
    const uint32_t raw = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t base = (raw + 127u) & ~127u;
    const uint32_t inB = base;                  // S input boxes
    const uint32_t outB = base + S * BOX;       // 2 output boxes
    const uint32_t bar = outB + 2 * BOX;        // S mbarriers
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nTiles = (uint32_t)p.nTiles;
    const uint32_t G = gridDim.x;
    const uint32_t t0 = blockIdx.x;
    if (t0 >= nTiles) return;
    const uint32_t nIt = (nTiles - t0 + G - 1) / G;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init_t(bar + 8u * s, 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // inits visible to the TMA unit
    }
    __syncthreads();
    int ci[5], co[5];
    if (tid == 0) {
        for (int s = 0; s < S && (uint32_t)s < nIt; ++s) {
            tma_coords(p, t0 + (uint32_t)s * G, ci, co);
            mbar_expect_tx(bar + 8u * s, BOX);
            tma_load<R>(inB + (uint32_t)s * BOX, &p.inMap, ci, bar + 8u * s);
        }
    }
    uint32_t stage = 0;
    for (uint32_t it = 0; it < nIt; ++it) {
        const uint32_t ob = outB + (it & 1u) * BOX;
        if (tid == 0)  // the store of iteration it-2 has read this output box
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        mbar_wait_t(bar + 8u * stage, (it / S) & 1u);
        // diagonal transpose: in[b][a] -> out[a][b], conflict-free both ways
        const uint32_t ib = inB + stage * BOX;
#pragma unroll 4
        for (int k = warp; k < (TA / 32) * TB; k += 8) {
            const int a = (k % (TA / 32)) * 32 + lane;
            const int b = (k / (TA / 32) + lane) % TB;
            const W v = lds<W>(ib + (uint32_t)(b * TA + a) * (uint32_t)sizeof(W));
            sts(ob + (uint32_t)(a * TB + b) * (uint32_t)sizeof(W), v);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
        __syncthreads();
        if (tid == 0) {
            tma_coords(p, t0 + it * G, ci, co);
            tma_store<R>(&p.outMap, co, ob);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            // every thread has read this input stage: refill it with tile it+S
            const uint32_t itn = it + S;
            if (itn < nIt) {
                tma_coords(p, t0 + itn * G, ci, co);
                mbar_expect_tx(bar + 8u * stage, BOX);
                tma_load<R>(ib, &p.inMap, ci, bar + 8u * stage);
            }
        }
        stage = (stage + 1 == (uint32_t)S) ? 0u : stage + 1;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA 2-D kernel: (word, TA, TB) in {(u32, 64, 64), (u64, 32, 64)}, 3 stages,
// tensor rank 2..5
const void* pick_tiled2d_tma(int esize, int rank) {
#define TT_TMA(W, TA, TB)                                                          \
    switch (rank) {                                                                \
        case 2: return (const void*)&tiled2d_tma_kernel<W, TA, TB, 3, 2>;         \
        case 3: return (const void*)&tiled2d_tma_kernel<W, TA, TB, 3, 3>;         \
        case 4: return (const void*)&tiled2d_tma_kernel<W, TA, TB, 3, 4>;         \
        case 5: return (const void*)&tiled2d_tma_kernel<W, TA, TB, 3, 5>;         \
        default: return nullptr;                                                   \
    }
    if (esize == 4) { TT_TMA(uint32_t, 64, 64) }
    if (esize == 8) { TT_TMA(uint64_t, 32, 64) }
    return nullptr;
#undef TT_TMA
}

}  // namespace tt
