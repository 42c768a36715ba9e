// hcb_dist.cu -- per-phase kernels of the 1D-partitioned multi-GPU solve
// (SURVEY.md §8(e)).
//
// Every rank owns a contiguous node range [lo, hi) (edge-balanced) and keeps a
// replicated copy of the solver's state word X[n] (hcb_solve.cu encoding:
// 0 / T / C|FBIT).  A round is
//   assign  (owned active nodes; X[u] = T; boundary nodes emit (u, T))
//   -> exchange + apply on every rank
//   resolve (owned active nodes; losers -> next owned worklist; winners set
//            FBIT and boundary winners emit (u, C|FBIT))
//   -> exchange + apply; all-reduce (|W'|, conflicts) drives the identical
//      mode decision / termination on every rank (driver.py:145-152).
// Only boundary nodes (a neighbour outside [lo, hi)) are exchanged: no other
// rank ever reads an interior node's word.  Round semantics are those of the
// single-GPU solve (reference coloring.py:113-176), so any partition gives
// the bit-identical coloring.
//
// Mapping: one warp per node, coalesced column loads, 64-bit color-mask mex
// with a 1024-color shared-memory window fallback.  These launch per phase
// because the exchange between phases is a collective.
#include "hcb_partition.cuh"

namespace hcb {
namespace dist {

constexpr int BLOCK = 256;
constexpr int NW = BLOCK / 32;
constexpr unsigned FBIT = 0x80000000u;
constexpr unsigned CMASK = 0x7fffffffu;
constexpr int WIN_WORDS = 32;

inline unsigned grid_for(long long items, int per_block) {
    long long g = (items + per_block - 1) / per_block;
    const long long cap = (long long)num_sms() * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// warp-aggregated append of (u, val) pairs
__device__ __forceinline__ void emit(bool want, int u, unsigned val, int *ids, unsigned *vals,
                                     unsigned long long *cnt) {
    const unsigned bal = __ballot_sync(FULL, want);
    if (!bal) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(cnt, (unsigned long long)__popc(bal));
    base = __shfl_sync(FULL, base, 0);
    if (want) {
        const unsigned long long pos = base + __popc(bal & lanemask_lt());
        ids[pos] = u;
        if (vals) vals[pos] = val;
    }
}

__device__ unsigned warp_mex(const long long *ro, const int *ci, const unsigned *X, int u, unsigned *bm) {
    const unsigned lane = lane_id();
    const long long b = ro[u], e = ro[u + 1];
    unsigned long long mask = 0;
    for (long long k = b + lane; k < e; k += 32) {
        const unsigned x = X[ci[k]];
        const unsigned c = x & CMASK;
        if ((x & FBIT) && c <= 64u) mask |= 1ull << (c - 1u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mask |= __shfl_xor_sync(FULL, mask, o);
    if (mask != ~0ull) return (unsigned)__ffsll((long long)~mask);
    const unsigned lim = (unsigned)(e - b) + 1u;  // mex <= deg+1 (_kernels.pyx:49)
    for (unsigned w0 = 64;; w0 += WIN_WORDS * 32) {
        bm[lane] = 0u;
        __syncwarp();
        const unsigned hi = min(lim, w0 + WIN_WORDS * 32);
        for (long long k = b + lane; k < e; k += 32) {
            const unsigned x = X[ci[k]];
            const unsigned c = x & CMASK;
            if ((x & FBIT) && c > w0 && c <= hi) atomicOr(&bm[(c - w0 - 1u) >> 5], 1u << ((c - w0 - 1u) & 31u));
        }
        __syncwarp();
        const unsigned word = bm[lane];
        const unsigned bal = __ballot_sync(FULL, word != FULL);
        __syncwarp();
        if (bal) {
            const int f = __ffs(bal) - 1;
            return w0 + (unsigned)f * 32u + (unsigned)__ffs(~__shfl_sync(FULL, word, f));
        }
    }
}

// node of work item i: list entry (data-driven) or lo + i (topology sweep)
__device__ __forceinline__ int item_node(const int *list, long long lo, long long i) {
    return list ? list[i] : (int)(lo + i);
}

__global__ void __launch_bounds__(BLOCK) assign_kernel(const long long *ro, const int *ci, unsigned *X,
                                                       const int *list, long long count, long long lo,
                                                       const unsigned char *boundary, int *out_ids,
                                                       unsigned *out_vals, unsigned long long *out_cnt) {
    __shared__ unsigned bm[NW][WIN_WORDS];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const long long nwarps = (long long)gridDim.x * NW;
    // iterate whole warps (32 items) so the warp-aggregated emit stays converged
    for (long long base = ((long long)blockIdx.x * NW + warp) * 32; base < count; base += nwarps * 32) {
        int mine = -1;
        unsigned mine_t = 0;
        for (int j = 0; j < 32 && base + j < count; ++j) {
            const int u = item_node(list, lo, base + j);
            const unsigned xu = X[u];
            if (!list && (xu & FBIT)) continue;  // topology sweep: inactive (_kernels.pyx:76-77)
            const unsigned T = warp_mex(ro, ci, X, u, bm[warp]);
            if (lane == 0) X[u] = T;
            if (lane == (unsigned)j) { mine = u; mine_t = T; }
        }
        emit(mine >= 0 && boundary[mine], mine, mine_t, out_ids, out_vals, out_cnt);
    }
}

__global__ void __launch_bounds__(BLOCK) resolve_kernel(const long long *ro, const int *ci, unsigned *X,
                                                        const int *list, long long count, long long lo,
                                                        const unsigned char *boundary, int *next,
                                                        unsigned long long *next_cnt, int *out_ids,
                                                        unsigned *out_vals, unsigned long long *out_cnt,
                                                        unsigned long long *conflicts) {
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const long long nwarps = (long long)gridDim.x * NW;
    unsigned long long my_conf = 0;
    for (long long base = ((long long)blockIdx.x * NW + warp) * 32; base < count; base += nwarps * 32) {
        int mine = -1;
        bool lost = false;
        unsigned win_val = 0;
        for (int j = 0; j < 32 && base + j < count; ++j) {
            const int u = item_node(list, lo, base + j);
            const unsigned xu = X[u];
            if (!list && (xu & FBIT)) continue;  // topology sweep: stamp != round (_kernels.pyx:135-136)
            unsigned cnt = 0;
            const long long b = ro[u], e = ro[u + 1];
            for (long long k0 = b; k0 < e; k0 += 32) {
                const long long k = k0 + lane;
                const int v = k < e ? ci[k] : 0x7fffffff;
                if (v < u) cnt += (X[v] & CMASK) == xu;
                if (__any_sync(FULL, v >= u)) break;  // adjacency sorted (graph.py:193-197)
            }
            cnt = warp_sum(cnt);
            if (lane == 0) {
                my_conf += cnt;
                if (!cnt) X[u] = xu | FBIT;
            }
            if (lane == (unsigned)j) {
                mine = u;
                lost = cnt != 0;
                win_val = xu | FBIT;
            }
        }
        emit(mine >= 0 && lost, mine, 0, next, nullptr, next_cnt);
        emit(mine >= 0 && !lost && boundary[mine], mine, win_val, out_ids, out_vals, out_cnt);
    }
    my_conf = warp_sum(my_conf);
    if (lane == 0 && my_conf) atomicAdd(conflicts, my_conf);
}

__global__ void apply_kernel(unsigned *X, const int *ids, const unsigned *vals, long long count) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        X[ids[i]] = vals[i];
}

__global__ void boundary_kernel(const long long *ro, const int *ci, long long lo, long long hi,
                                unsigned char *flags) {
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const long long nwarps = (long long)gridDim.x * NW;
    for (long long u = lo + (long long)blockIdx.x * NW + warp; u < hi; u += nwarps) {
        bool out = false;
        for (long long k = ro[u] + lane; k < ro[u + 1] && !out; k += 32) {
            const long long v = ci[k];
            out = v < lo || v >= hi;
        }
        out = __any_sync(FULL, out);
        if (lane == 0) flags[u - lo] = out ? 1 : 0;
    }
}

__global__ void gather_colors_kernel(const unsigned *X, long long lo, long long hi, long long *colors) {
    for (long long u = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; u < hi;
         u += (long long)gridDim.x * blockDim.x)
        colors[u - lo] = (long long)(X[u] & CMASK);
}

}  // namespace dist
}  // namespace hcb

using namespace hcb;
using namespace hcb::dist;

extern "C" {

int hc_dist_boundary(const int64_t *d_ro, const int32_t *d_ci, int64_t lo, int64_t hi, uint8_t *d_flags,
                     void *stream) {
    HC_REQUIRE(lo >= 0 && hi >= lo, HC_ERR_INVALID, "dist_boundary: bad range");
    if (hi == lo) return HC_OK;
    boundary_kernel<<<grid_for(hi - lo, NW), BLOCK, 0, as_stream(stream)>>>((const long long *)d_ro, d_ci, lo, hi,
                                                                          d_flags);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_dist_assign(const int64_t *d_ro, const int32_t *d_ci, uint32_t *d_X, const int32_t *d_list,
                   int64_t count, int64_t lo, const uint8_t *d_boundary_rel, int32_t *d_out_ids,
                   uint32_t *d_out_vals, int64_t *d_out_cnt, void *stream) {
    HC_REQUIRE(count >= 0 && d_out_cnt, HC_ERR_INVALID, "dist_assign: bad arguments");
    if (count == 0) return HC_OK;
    // boundary flags are relative to lo; shift the pointer so boundary[u] works
    const unsigned char *bnd = d_boundary_rel - lo;
    assign_kernel<<<grid_for(count, NW * 32), BLOCK, 0, as_stream(stream)>>>(
        (const long long *)d_ro, d_ci, d_X, d_list, count, lo, bnd, d_out_ids, d_out_vals,
        (unsigned long long *)d_out_cnt);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_dist_resolve(const int64_t *d_ro, const int32_t *d_ci, uint32_t *d_X, const int32_t *d_list,
                    int64_t count, int64_t lo, const uint8_t *d_boundary_rel, int32_t *d_next,
                    int64_t *d_next_cnt, int32_t *d_out_ids, uint32_t *d_out_vals, int64_t *d_out_cnt,
                    int64_t *d_conflicts, void *stream) {
    HC_REQUIRE(count >= 0 && d_next_cnt && d_out_cnt && d_conflicts, HC_ERR_INVALID,
               "dist_resolve: bad arguments");
    if (count == 0) return HC_OK;
    const unsigned char *bnd = d_boundary_rel - lo;
    resolve_kernel<<<grid_for(count, NW * 32), BLOCK, 0, as_stream(stream)>>>(
        (const long long *)d_ro, d_ci, d_X, d_list, count, lo, bnd, d_next,
        (unsigned long long *)d_next_cnt, d_out_ids, d_out_vals, (unsigned long long *)d_out_cnt,
        (unsigned long long *)d_conflicts);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_dist_apply(uint32_t *d_X, const int32_t *d_ids, const uint32_t *d_vals, int64_t count, void *stream) {
    HC_REQUIRE(count >= 0, HC_ERR_INVALID, "dist_apply: bad count");
    if (count == 0) return HC_OK;
    apply_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(d_X, d_ids, d_vals, count);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_dist_colors(const uint32_t *d_X, int64_t lo, int64_t hi, int64_t *d_colors, void *stream) {
    HC_REQUIRE(hi >= lo, HC_ERR_INVALID, "dist_colors: bad range");
    if (hi == lo) return HC_OK;
    gather_colors_kernel<<<grid_for(hi - lo, 256), 256, 0, as_stream(stream)>>>(d_X, lo, hi,
                                                                               (long long *)d_colors);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

}  // extern "C"
