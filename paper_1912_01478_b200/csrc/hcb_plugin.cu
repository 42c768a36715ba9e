// hcb_plugin.cu -- the reference's kernel-module plugin API on the device.
//
// One entry point per function of pkg/src/hybridcolor/_kernels.pyx:25-187,
// same argument meaning, int64 device arrays exactly as the reference passes
// them (coloring.py:127-139, 160-173; bench.py:86-92).  These are the per-round
// operators a `cuda` backend registered in hybridcolor._backend._BACKENDS
// (_backend.py:15-21) would call; the product solve (hcb_solve.cu) fuses the
// whole round loop instead.
//
// Mapping: one warp per processed node.  The assign mex is computed over a
// 1024-color shared-memory bitmap window per warp, sliding the window until a
// free color is found, so any degree is handled (the reference tracks only
// colors 1..deg+1, _kernels.pyx:49-56; colors above deg+1 can never be the mex,
// so ignoring them is equivalent).  Resolve counts every lower-id neighbour
// with the same stamped color (_kernels.pyx:110-113) without assuming sorted
// rows, because CsrGraph(...) built by hand is not validated (graph.py:49-67).
// Pushes go through one relaxed atomicAdd on the shared cursor and are dropped
// past `capacity` exactly like hc_fetch_add + `if pos < cap` (_kernels.pyx:16-23,
// 116-118).
#include "hcb_partition.cuh"

namespace hcb {
namespace plugin {

constexpr int BLOCK = 256;
constexpr int NW = BLOCK / 32;
constexpr int WIN_WORDS = 32;  // 1024 colors per window pass

__device__ __forceinline__ void assign_one(const long long *ro, const long long *ci,
                                           const long long *cr, long long *cw, long long *stamp,
                                           long long u, long long round_no, unsigned *bm) {
    const unsigned lane = lane_id();
    const long long b = ro[u], e = ro[u + 1];
    const long long lim = e - b + 1;
    for (long long w0 = 0;; w0 += WIN_WORDS * 32) {
        bm[lane] = 0u;
        __syncwarp();
        const long long hi = min(lim, w0 + WIN_WORDS * 32);
        for (long long k = b + lane; k < e; k += 32) {
            const long long c = cr[ci[k]];
            if (c > w0 && c <= hi) {
                const long long bit = c - w0 - 1;
                atomicOr(&bm[bit >> 5], 1u << (bit & 31));
            }
        }
        __syncwarp();
        const unsigned word = bm[lane];
        const unsigned bal = __ballot_sync(FULL, word != FULL);
        __syncwarp();
        if (bal) {
            const int f = __ffs(bal) - 1;
            const unsigned fw = __shfl_sync(FULL, word, f);
            if (lane == 0) {
                cw[u] = w0 + (long long)f * 32 + __ffs(~fw);
                stamp[u] = round_no;
            }
            return;
        }
    }
}

__global__ void __launch_bounds__(BLOCK) assign_list_kernel(const long long *ro, const long long *ci,
                                                            const long long *cr, long long *cw,
                                                            long long *stamp, const long long *nodes,
                                                            long long m, long long round_no) {
    __shared__ unsigned bm[NW][WIN_WORDS];
    const long long w = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * BLOCK) >> 5;
    for (long long i = w; i < m; i += nwarps)
        assign_one(ro, ci, cr, cw, stamp, nodes[i], round_no, bm[threadIdx.x >> 5]);
}

__global__ void __launch_bounds__(BLOCK) assign_sweep_kernel(const long long *ro, const long long *ci,
                                                             const long long *cr, long long *cw,
                                                             long long *stamp, long long n,
                                                             long long round_no,
                                                             unsigned long long *acc) {
    __shared__ unsigned bm[NW][WIN_WORDS];
    const long long w = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * BLOCK) >> 5;
    unsigned long long processed = 0;
    for (long long u = w; u < n; u += nwarps) {
        if (cr[u] == 0) {  // activity test, _kernels.pyx:76-77
            assign_one(ro, ci, cr, cw, stamp, u, round_no, bm[threadIdx.x >> 5]);
            ++processed;
        }
    }
    if (lane_id() == 0 && processed) atomicAdd(acc, processed);
}

__device__ __forceinline__ unsigned long long resolve_one(const long long *ro, const long long *ci,
                                                          const long long *cr, long long *cw,
                                                          const long long *stamp, long long u,
                                                          long long round_no, long long *next_ids,
                                                          long long cap, unsigned long long *cursor) {
    const unsigned lane = lane_id();
    const long long cu = cr[u];
    unsigned long long cnt = 0;
    for (long long k = ro[u] + lane; k < ro[u + 1]; k += 32) {
        const long long v = ci[k];
        if (v < u && stamp[v] == round_no && cr[v] == cu) ++cnt;
    }
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt > 0) {
        cw[u] = 0;
        const unsigned long long pos = atomicAdd(cursor, 1ull);
        if ((long long)pos < cap) next_ids[pos] = u;
    }
    return cnt;
}

__global__ void __launch_bounds__(BLOCK) resolve_list_kernel(
    const long long *ro, const long long *ci, const long long *cr, long long *cw,
    const long long *stamp, const long long *nodes, long long m, long long round_no,
    long long *next_ids, long long cap, unsigned long long *cursor, unsigned long long *acc) {
    const long long w = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * BLOCK) >> 5;
    unsigned long long conflicts = 0;
    for (long long i = w; i < m; i += nwarps)
        conflicts += resolve_one(ro, ci, cr, cw, stamp, nodes[i], round_no, next_ids, cap, cursor);
    if (lane_id() == 0 && conflicts) atomicAdd(acc, conflicts);
}

__global__ void __launch_bounds__(BLOCK) resolve_sweep_kernel(
    const long long *ro, const long long *ci, const long long *cr, long long *cw,
    const long long *stamp, long long n, long long round_no, long long *next_ids, long long cap,
    unsigned long long *cursor, unsigned long long *acc) {
    const long long w = ((long long)blockIdx.x * BLOCK + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * BLOCK) >> 5;
    unsigned long long conflicts = 0;
    for (long long u = w; u < n; u += nwarps)
        if (stamp[u] == round_no)  // activity test, _kernels.pyx:135-136
            conflicts += resolve_one(ro, ci, cr, cw, stamp, u, round_no, next_ids, cap, cursor);
    if (lane_id() == 0 && conflicts) atomicAdd(acc, conflicts);
}

// bench kernels (_kernels.pyx:152-187): thread per node, warp-aggregated push
__device__ __forceinline__ void bench_node(long long u, bool live, unsigned char *active,
                                           long long cutoff, long long *next_ids, long long cap,
                                           unsigned long long *cursor) {
    bool push = false;
    if (live) {
        if (u <= cutoff) active[u] = 0;
        else push = true;
    }
    const unsigned bal = __ballot_sync(FULL, push);
    if (!bal) return;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(cursor, (unsigned long long)__popc(bal));
    base = __shfl_sync(FULL, base, 0);
    if (push) {
        const long long pos = (long long)(base + __popc(bal & lanemask_lt()));
        if (pos < cap) next_ids[pos] = u;
    }
}

__global__ void __launch_bounds__(BLOCK) bench_list_kernel(const long long *nodes, long long m,
                                                           unsigned char *active, long long cutoff,
                                                           long long *next_ids, long long cap,
                                                           unsigned long long *cursor) {
    const long long stride = (long long)gridDim.x * BLOCK;
    const long long span = (m + 31) / 32 * 32;  // whole warps stay converged for the ballot
    for (long long i = (long long)blockIdx.x * BLOCK + threadIdx.x; i < span; i += stride) {
        const bool live = i < m;
        bench_node(live ? nodes[i] : 0, live, active, cutoff, next_ids, cap, cursor);
    }
}

__global__ void __launch_bounds__(BLOCK) bench_sweep_kernel(unsigned char *active, long long n,
                                                            long long cutoff, long long *next_ids,
                                                            long long cap,
                                                            unsigned long long *cursor) {
    const long long stride = (long long)gridDim.x * BLOCK;
    const long long span = (n + 31) / 32 * 32;
    for (long long u = (long long)blockIdx.x * BLOCK + threadIdx.x; u < span; u += stride) {
        const bool live = u < n && active[u] != 0;
        bench_node(u, live, active, cutoff, next_ids, cap, cursor);
    }
}

// commits between phases (coloring.py:105-110)
__global__ void commit_list_kernel(long long *cr, const long long *cw, const long long *nodes,
                                   long long m) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        const long long u = nodes[i];
        cr[u] = cw[u];
    }
}

__global__ void commit_stamped_kernel(long long *cr, const long long *cw, const long long *stamp,
                                      long long n, long long round_no) {
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (long long)gridDim.x * blockDim.x)
        if (stamp[u] == round_no) cr[u] = cw[u];
}

// ---------------------------------------------------------------- wl sort
__global__ void wl_mark_kernel(const long long *next, long long m, long long cap, unsigned *flags,
                               unsigned *status) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        const long long id = next[i];
        if (id < 0 || id >= cap) {
            atomicOr(status, 2u);
            continue;
        }
        if (atomicAdd(&flags[id], 1u) != 0u) atomicOr(status, 1u);
    }
}

struct FlagBin {
    const unsigned *flags;
    __device__ int operator()(long long i) const { return flags[i] ? 0 : -1; }
};
struct EmitI64 {
    __device__ long long operator()(long long i) const { return i; }
};

inline unsigned grid_for(long long items, int per_block_items) {
    long long g = (items + per_block_items - 1) / per_block_items;
    const long long cap = (long long)num_sms() * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace plugin
}  // namespace hcb

using namespace hcb;
using namespace hcb::plugin;

static int read_acc(int64_t *d_acc, int64_t *h_out, cudaStream_t st) {
    if (!h_out) return HC_OK;
    HC_CUDA_TRY(cudaMemcpyAsync(h_out, d_acc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    return HC_OK;
}

extern "C" {

int hc_k_assign_from_list(const int64_t *ro, const int64_t *ci, const int64_t *cr, int64_t *cw,
                          int64_t *stamp, const int64_t *nodes, int64_t m, int64_t round_no,
                          int64_t max_degree, void *stream) {
    (void)max_degree;  // scratch sizing only in the reference (_kernels.pyx:40)
    HC_REQUIRE(m >= 0, HC_ERR_INVALID, "assign_from_list: negative list length");
    if (m == 0) return HC_OK;  // _kernels.pyx:36-37
    cudaStream_t st = as_stream(stream);
    assign_list_kernel<<<grid_for(m, NW), BLOCK, 0, st>>>(
        (const long long *)ro, (const long long *)ci, (const long long *)cr, (long long *)cw,
        (long long *)stamp, (const long long *)nodes, m, round_no);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_k_assign_sweep(const int64_t *ro, const int64_t *ci, const int64_t *cr, int64_t *cw,
                      int64_t *stamp, int64_t n, int64_t round_no, int64_t max_degree,
                      int64_t *d_acc, int64_t *h_processed, void *stream) {
    (void)max_degree;
    HC_REQUIRE(n >= 0 && d_acc, HC_ERR_INVALID, "assign_sweep: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (n > 0) {
        assign_sweep_kernel<<<grid_for(n, NW), BLOCK, 0, st>>>(
            (const long long *)ro, (const long long *)ci, (const long long *)cr, (long long *)cw,
            (long long *)stamp, n, round_no, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    return read_acc(d_acc, h_processed, st);
}

int hc_k_resolve_from_list(const int64_t *ro, const int64_t *ci, const int64_t *cr, int64_t *cw,
                           const int64_t *stamp, const int64_t *nodes, int64_t m, int64_t round_no,
                           int64_t *next_ids, int64_t cap, int64_t *cursor, int64_t *d_acc,
                           int64_t *h_conflicts, void *stream) {
    HC_REQUIRE(m >= 0 && cap >= 0 && d_acc && cursor, HC_ERR_INVALID,
               "resolve_from_list: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (m > 0) {
        resolve_list_kernel<<<grid_for(m, NW), BLOCK, 0, st>>>(
            (const long long *)ro, (const long long *)ci, (const long long *)cr, (long long *)cw,
            (const long long *)stamp, (const long long *)nodes, m, round_no, (long long *)next_ids,
            cap, (unsigned long long *)cursor, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    return read_acc(d_acc, h_conflicts, st);
}

int hc_k_resolve_sweep(const int64_t *ro, const int64_t *ci, const int64_t *cr, int64_t *cw,
                       const int64_t *stamp, int64_t n, int64_t round_no, int64_t *next_ids,
                       int64_t cap, int64_t *cursor, int64_t *d_acc, int64_t *h_conflicts,
                       void *stream) {
    HC_REQUIRE(n >= 0 && cap >= 0 && d_acc && cursor, HC_ERR_INVALID, "resolve_sweep: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (n > 0) {
        resolve_sweep_kernel<<<grid_for(n, NW), BLOCK, 0, st>>>(
            (const long long *)ro, (const long long *)ci, (const long long *)cr, (long long *)cw,
            (const long long *)stamp, n, round_no, (long long *)next_ids, cap,
            (unsigned long long *)cursor, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    return read_acc(d_acc, h_conflicts, st);
}

int hc_k_bench_from_list(const int64_t *nodes, int64_t m, uint8_t *active, int64_t cutoff,
                         int64_t *next_ids, int64_t cap, int64_t *cursor, void *stream) {
    HC_REQUIRE(m >= 0 && cap >= 0 && cursor, HC_ERR_INVALID, "bench_from_list: bad arguments");
    if (m == 0) return HC_OK;
    cudaStream_t st = as_stream(stream);
    bench_list_kernel<<<grid_for(m, BLOCK), BLOCK, 0, st>>>((const long long *)nodes, m, active,
                                                            cutoff, (long long *)next_ids, cap,
                                                            (unsigned long long *)cursor);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_k_bench_sweep(uint8_t *active, int64_t n, int64_t cutoff, int64_t *next_ids, int64_t cap,
                     int64_t *cursor, void *stream) {
    HC_REQUIRE(n >= 0 && cap >= 0 && cursor, HC_ERR_INVALID, "bench_sweep: bad arguments");
    if (n == 0) return HC_OK;
    cudaStream_t st = as_stream(stream);
    bench_sweep_kernel<<<grid_for(n, BLOCK), BLOCK, 0, st>>>(active, n, cutoff,
                                                             (long long *)next_ids, cap,
                                                             (unsigned long long *)cursor);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_k_commit_list(int64_t *cr, const int64_t *cw, const int64_t *nodes, int64_t m, void *stream) {
    HC_REQUIRE(m >= 0, HC_ERR_INVALID, "commit_list: negative length");
    if (m == 0) return HC_OK;
    commit_list_kernel<<<grid_for(m, 256), 256, 0, as_stream(stream)>>>(
        (long long *)cr, (const long long *)cw, (const long long *)nodes, m);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_k_commit_stamped(int64_t *cr, const int64_t *cw, const int64_t *stamp, int64_t n,
                        int64_t round_no, void *stream) {
    HC_REQUIRE(n >= 0, HC_ERR_INVALID, "commit_stamped: negative length");
    if (n == 0) return HC_OK;
    commit_stamped_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(
        (long long *)cr, (const long long *)cw, (const long long *)stamp, n, round_no);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

size_t hc_wl_sort_workspace_bytes(int64_t capacity) {
    if (capacity < 0) capacity = 0;
    return align_up(sizeof(unsigned) * (size_t)capacity, 256) + 256 +
           part_scratch_bytes(1, capacity);
}

int hc_wl_swap_and_sort(const int64_t *d_next, const int64_t *d_cursor, int64_t cap,
                        int64_t *d_sorted, int64_t *h_count, void *d_ws, size_t ws_bytes,
                        void *stream) {
    HC_REQUIRE(cap >= 0 && d_cursor && h_count, HC_ERR_INVALID, "swap_and_sort: bad arguments");
    HC_REQUIRE(d_ws && ws_bytes >= hc_wl_sort_workspace_bytes(cap), HC_ERR_WORKSPACE,
               "swap_and_sort: workspace too small");
    cudaStream_t st = as_stream(stream);
    int64_t m = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&m, d_cursor, sizeof m, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    *h_count = m;
    HC_REQUIRE(m <= cap, HC_ERR_WL_OVERFLOW, "worklist overflow: %lld pushes into capacity %lld",
               (long long)m, (long long)cap);  // worklist.py:79-83
    if (m == 0) return HC_OK;
    char *ws = reinterpret_cast<char *>(d_ws);
    unsigned *flags = reinterpret_cast<unsigned *>(ws);
    unsigned *status = reinterpret_cast<unsigned *>(ws + align_up(sizeof(unsigned) * (size_t)cap, 256));
    void *scratch = ws + align_up(sizeof(unsigned) * (size_t)cap, 256) + 256;
    HC_CUDA_TRY(cudaMemsetAsync(ws, 0, align_up(sizeof(unsigned) * (size_t)cap, 256) + 256, st));
    wl_mark_kernel<<<grid_for(m, 256), 256, 0, st>>>((const long long *)d_next, m, cap, flags, status);
    HC_CHECK_LAUNCH();
    int rc = ordered_partition<1>(cap, FlagBin{flags}, EmitI64{}, (long long *)d_sorted, scratch,
                                  nullptr, st);
    if (rc != HC_OK) return rc;
    unsigned h_status = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&h_status, status, sizeof h_status, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    HC_REQUIRE(!(h_status & 2u), HC_ERR_INVALID, "swap_and_sort: pushed id outside [0, capacity)");
    HC_REQUIRE(!(h_status & 1u), HC_ERR_DUPLICATE, "duplicate id pushed within one iteration");
    return HC_OK;
}

}  // extern "C"
