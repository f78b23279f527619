// common.cuh -- sm_100a helpers shared by the LP kernels.
//
// 1-D bulk TMA (cp.async.bulk) global<->shared copies completed on mbarriers,
// compile-time-aligned vector row loads, warp reductions.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cstdlib>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

// Checked build (-D TVLP_CHECKED=1, `python -m paper_2406_05128_b200.build
// --define TVLP_CHECKED=1 --out variants/checked/libtvlp_b200.so`): device-side
// bounds and protocol assertions on the index arithmetic of the hand-written
// kernels (staged spans, stage slots, unit/sub-chunk/row ranges, output
// offsets).  A failed assertion prints its site and traps the kernel.  The
// stand-in for compute-sanitizer on GPU pools where it is unavailable
// (tools/checked_tests.sh runs the GPU suite against this build).
#ifndef TVLP_CHECKED
#define TVLP_CHECKED 0
#endif
#if TVLP_CHECKED
#define TVLP_ASSERT(c)                                                                        \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("TVLP_ASSERT %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,   \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define TVLP_ASSERT(c) ((void)0)
#endif

namespace tvlp {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ---------------------------------------------------------------- bulk TMA
// global -> shared, completion signalled as tx bytes on `bar`.
// src, dst and bytes must be multiples of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 2-D tiled tensor copies (CUtensorMap passed as a __grid_constant__ kernel
// parameter).  smem boxes must be 128-byte aligned; out-of-bounds elements of
// a load box are zero-filled, out-of-bounds elements of a store box are
// skipped.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1,
                                             const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     map),
                 "r"(c0), "r"(c1), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// shared -> global, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Order generic-proxy shared-memory WRITES before subsequent async-proxy (TMA
// store) reads of them.  Not needed to recycle a buffer that was only READ by
// generic loads (write-after-read): the loaded values have been consumed
// before the refill is issued.  The fence also waits for this thread's
// outstanding memory operations, so it is kept off the serial carry chains.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- warp utils
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// round `bytes` up to 16 and make (bytes/16) odd: per-lane slot strides with an
// odd number of 16-byte granules keep 8 consecutive lanes' 16-B accesses in
// distinct bank groups.
constexpr int odd16_stride(int bytes) {
    int b = (bytes + 15) / 16 * 16;
    return ((b / 16) % 2 == 0) ? b + 16 : b;
}
constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int clcm(int a, int b) { return a / cgcd(a, b) * b; }

// ---------------------------------------------------------------- row loads
// Load M consecutive T values from shared memory at `p` into registers, using
// the widest vector accesses the compile-time alignment OFF (= address mod 16)
// allows.
template <typename T, int M, int I, int OFF>
struct RowLoad {
    static __device__ __forceinline__ void run(const T* p, T* a) {
        if constexpr (I < M) {
            constexpr int off = (OFF + I * (int)sizeof(T)) & 15;
            if constexpr (sizeof(T) == 4 && off == 0 && I + 4 <= M) {
                float4 v = *reinterpret_cast<const float4*>(p + I);
                a[I] = v.x;
                a[I + 1] = v.y;
                a[I + 2] = v.z;
                a[I + 3] = v.w;
                RowLoad<T, M, I + 4, OFF>::run(p, a);
            } else if constexpr (sizeof(T) == 4 && (off & 7) == 0 && I + 2 <= M) {
                float2 v = *reinterpret_cast<const float2*>(p + I);
                a[I] = v.x;
                a[I + 1] = v.y;
                RowLoad<T, M, I + 2, OFF>::run(p, a);
            } else if constexpr (sizeof(T) == 8 && off == 0 && I + 2 <= M) {
                double2 v = *reinterpret_cast<const double2*>(p + I);
                a[I] = v.x;
                a[I + 1] = v.y;
                RowLoad<T, M, I + 2, OFF>::run(p, a);
            } else {
                a[I] = p[I];
                RowLoad<T, M, I + 1, OFF>::run(p, a);
            }
        }
    }
};
template <typename T, int M, int OFF>
__device__ __forceinline__ void load_row(const T* p, T (&a)[M]) {
    RowLoad<T, M, 0, OFF>::run(p, a);
}

// Same, with the alignment given as a value that is a compile-time constant
// after loop unrolling (the switch folds away).
template <typename T, int M>
__device__ __forceinline__ void load_row_at(const T* p, T (&a)[M], int off) {
    switch (off & 15) {
        case 0: load_row<T, M, 0>(p, a); break;
        case 4: load_row<T, M, 4>(p, a); break;
        case 8: load_row<T, M, 8>(p, a); break;
        default: load_row<T, M, 12>(p, a); break;
    }
}

// compile-time loop: f(std::integral_constant<int, I>{}) for I = 0..N-1
template <int I, int N, typename F>
__device__ __forceinline__ void static_for_impl(F&& f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for_impl<I + 1, N>(f);
    }
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl<0, N>(f);
}

template <typename T>
__device__ __forceinline__ bool is_finite_val(T x) {
    return isfinite(x);
}


// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialization, so its
// launch (block scheduling, prologue) overlaps the tail of the previous
// kernel in the stream; griddepcontrol.wait then blocks until that kernel has
// completed and its writes are visible.  Kernels call it before touching
// global memory.  Without the launch attribute the wait is a no-op.
// TVLP_PDL_TRIGGER=1 also triggers the dependent right after the wait
// (griddepcontrol.launch_dependents), so the next kernel's CTAs park in their
// own wait on the SMs this grid's finished CTAs free.  Measured slower on
// every config (config 3: 340 -> 352 us, config 1: 138 -> 166 us): the parked
// CTAs hold SM slots through this grid's tail.  Off by default.
#ifndef TVLP_PDL_TRIGGER
#define TVLP_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
#if TVLP_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("TVLP_PDL");
        return v == nullptr || v[0] != '0';
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace tvlp
