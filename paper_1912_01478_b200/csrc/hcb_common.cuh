// hcb_common.cuh -- shared helpers for libhcb.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/hcb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libhcb targets sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace hcb {

// last error message per host thread (hc_last_error)
void set_error(const char *fmt, ...);

#define HC_CUDA_TRY(expr)                                                             \
    do {                                                                              \
        cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            ::hcb::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                             __FILE__, __LINE__);                                     \
            return HC_ERR_CUDA;                                                       \
        }                                                                             \
    } while (0)

#define HC_CHECK_LAUNCH() HC_CUDA_TRY(cudaGetLastError())

#define HC_REQUIRE(cond, code, ...)           \
    do {                                      \
        if (!(cond)) {                        \
            ::hcb::set_error(__VA_ARGS__);    \
            return (code);                    \
        }                                     \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int num_sms();

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// system-scope accesses for the cross-GPU mailboxes (peer memory over NVLink)
__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// inclusive warp scan
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const unsigned lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, v, o);
        if (lane >= (unsigned)o) v += y;
    }
    return v;
}

// Software grid barrier for a co-resident (cooperatively launched) grid.
// Sense is a monotonically increasing generation; the last arriver resets the
// count and bumps the generation with release semantics.  The gpu-scope fences
// also invalidate the SM's L1 so the next phase reads fresh global state.
struct GridBarrier {
    unsigned count;
    unsigned gen;
};

#ifndef HC_FAST_BARRIER
#define HC_FAST_BARRIER 1
#endif
#ifndef HC_BAR_SLEEP
#define HC_BAR_SLEEP 20  // ns between polls of the barrier generation
#endif
__device__ __forceinline__ void grid_sync(GridBarrier *b, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
#if HC_FAST_BARRIER
        // arrival is one acq_rel atomic (releases the CTA's writes, ordered
        // before it by the CTA barrier); the last arriver resets the count and
        // publishes the next generation with a release store; the waiters'
        // acquire load of it orders (and L1-invalidates) what follows
        const unsigned g = *(volatile unsigned *)&b->gen;
        unsigned arrived;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(&b->count) : "memory");
        if (arrived == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&b->count), "r"(0u) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&b->gen), "r"(g + 1u) : "memory");
        } else {
            while (ld_acquire_u32(&b->gen) == g) __nanosleep(HC_BAR_SLEEP);
        }
#else
        unsigned g = ld_acquire_u32(&b->gen);
        __threadfence();
        unsigned arrived = atomicAdd(&b->count, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(&b->count, 0u);
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (ld_acquire_u32(&b->gen) == g) __nanosleep(20);
        }
        __threadfence();
#endif
    }
    __syncthreads();
}

}  // namespace hcb
