// hcb_pushbench.cu -- the paper's §3 micro-benchmark pair on the device
// (reference pkg/src/hybridcolor/bench.py:67-161, kernels _kernels.pyx:152-187;
// PAPER.md:125-165).
//
// Both variants deactivate, every iteration, the `batch` lowest-id active
// nodes and push every other active node to the next worklist:
//   push_wl   (data-driven)     walks the current worklist
//   push_nowl (topology-driven) sweeps all ids testing the active flag,
//                               still maintaining the worklist
// The whole pipe runs in ONE persistent cooperative kernel.  The worklist is
// kept sorted without a sort: CTA b processes a contiguous share of its input
// (list positions for push_wl, ids for push_nowl) and compacts the survivors
// order-preservingly into output segment b; the next iteration rebuilds the
// segment prefix.  The cutoff (bench.py:80: the take-th smallest active id) is
// read from the sorted list.  Per iteration the device records the push
// phase's %globaltimer duration (bench.py:85-92 times the kernel only), the
// worklist size and the cutoff; the deactivated set of iteration t is then
// exactly the id range (cutoff[t-1], cutoff[t]].
#include "hcb_partition.cuh"

namespace hcb {
namespace pushbench {

constexpr int BLOCK = 512;
constexpr int NW = BLOCK / 32;
constexpr int MAXG = 512;  // max CTAs (segments)
constexpr int EPT = 8;     // elements per thread per tile
static_assert(EPT * NW % 32 == 0, "scan layout");

struct Ctrl {
    GridBarrier bar;
    long long iters;
    long long overflow;
    unsigned segcnt[2][MAXG];
};

struct Params {
    long long n;
    long long batch;
    int variant;  // 0 push_wl, 1 push_nowl
    unsigned char *active;
    int *seg[2];  // segmented lists, capacity segcap per CTA
    long long segcap;
    Ctrl *ctrl;
    long long *rec_ns, *rec_size, *rec_cutoff;
    long long max_iters;
    unsigned nblocks;
};

struct Smem {
    unsigned prefix[MAXG + 1];
    unsigned warp_tmp[NW];
    unsigned jw[EPT * NW];
    unsigned tot;
    long long cutoff;
};

// element v of the current list (dense identity in iteration 0)
__device__ __forceinline__ int list_at(const Params &P, const Smem &sm, int p, bool dense, unsigned long long v,
                                       unsigned &s) {
    if (dense) return (int)v;
    while (sm.prefix[s + 1] <= v) ++s;
    const int *cur = p ? P.seg[1] : P.seg[0];  // select, not a runtime-indexed param array
    return cur[(long long)s * P.segcap + (long long)(v - sm.prefix[s])];
}

__device__ __forceinline__ unsigned seg_of(const Smem &sm, unsigned nseg, unsigned long long v) {
    unsigned lo = 0, hi = nseg;
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (sm.prefix[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// block exclusive sum of one value per thread; *total = sum
__device__ __forceinline__ unsigned block_excl_sum(unsigned x, unsigned &total, Smem &sm) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const unsigned incl = warp_incl_scan(x);
    if (lane == 31) sm.warp_tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned v = lane < NW ? sm.warp_tmp[lane] : 0u;
        const unsigned vi = warp_incl_scan(v);
        if (lane < NW) sm.warp_tmp[lane] = vi - v;
        if (lane == 31) sm.tot = vi;
    }
    __syncthreads();
    const unsigned r = sm.warp_tmp[warp] + incl - x;
    total = sm.tot;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(BLOCK, 2) pushbench_kernel(Params P) {
    __shared__ Smem sm;
    Ctrl *C = P.ctrl;
    const unsigned G = P.nblocks;
    for (long long u = (long long)blockIdx.x * BLOCK + threadIdx.x; u < P.n; u += (long long)G * BLOCK)
        P.active[u] = 1;
    grid_sync(&C->bar, G);
    unsigned long long t0 = 0;
    long long it = 0;
    for (;; ++it) {
        const int p = (int)(it & 1), np = p ^ 1;
        const bool dense = it == 0;
        // ---- current worklist: segment prefix of the previous output
        unsigned long long size;
        if (dense) {
            size = (unsigned long long)P.n;
        } else {
            for (unsigned s = threadIdx.x; s < G; s += BLOCK) sm.prefix[s + 1] = __ldcg(&C->segcnt[p][s]);
            if (threadIdx.x == 0) sm.prefix[0] = 0;
            __syncthreads();
            if (threadIdx.x == 0)  // G <= 512 values: a serial scan by one thread is plenty
                for (unsigned s = 1; s <= G; ++s) sm.prefix[s] += sm.prefix[s - 1];
            __syncthreads();
            size = sm.prefix[G];
        }
        if (size == 0) break;  // pipe drained (bench.py:77)
        // ---- cutoff: the take-th smallest active id (bench.py:79-80)
        if (threadIdx.x == 0) {
            const unsigned long long take = min((unsigned long long)P.batch, size);
            unsigned s = dense ? 0u : seg_of(sm, G, take - 1);
            sm.cutoff = list_at(P, sm, p, dense, take - 1, s);
        }
        __syncthreads();
        const long long cutoff = sm.cutoff;
        grid_sync(&C->bar, G);
        if (blockIdx.x == 0 && threadIdx.x == 0) t0 = globaltimer();
        // ---- timed push phase
        const unsigned long long span = P.variant == 0 ? size : (unsigned long long)P.n;
        // CTA shares rounded to 16 elements (aligned 16-byte flag loads)
        const unsigned long long lo = blockIdx.x == 0 ? 0 : ((span * blockIdx.x / G) & ~15ull);
        const unsigned long long hi = blockIdx.x + 1 == G ? span : ((span * (blockIdx.x + 1) / G) & ~15ull);
        int *out = (np ? P.seg[1] : P.seg[0]) + (long long)blockIdx.x * P.segcap;
        unsigned written = 0;
        {
            // element v = base + j*BLOCK + tid: coalesced reads of the flags
            // (push_nowl) or the list (push_wl), coalesced j-major
            // order-preserving compaction of the survivors
            const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
            const bool wl = P.variant == 0;
            unsigned s = (wl && !dense) ? seg_of(sm, G, lo < size ? lo : 0) : 0u;
            for (unsigned long long base = lo; base < hi; base += (unsigned long long)BLOCK * EPT) {
                int ids[EPT];
                unsigned bal[EPT];
                // all EPT loads first (independent), then decide
#pragma unroll
                for (int j = 0; j < EPT; ++j) {
                    const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
                    ids[j] = -1;
                    if (v < hi) {
                        if (wl) ids[j] = list_at(P, sm, p, dense, v, s);     // bench_from_list
                        else ids[j] = P.active[v] ? (int)v : -1;              // bench_sweep
                    }
                }
#pragma unroll
                for (int j = 0; j < EPT; ++j) {
                    bool keep = false;
                    if (ids[j] >= 0) {
                        if (ids[j] <= cutoff) P.active[ids[j]] = 0;  // _kernels.pyx:159-160 / 178-179
                        else keep = true;                            // push (_kernels.pyx:161-165)
                    }
                    bal[j] = __ballot_sync(FULL, keep);
                }
                // tiles without survivors (the deactivated prefix in push_nowl
                // sweeps) skip the compaction: one barrier instead of three
                unsigned any = 0;
#pragma unroll
                for (int j = 0; j < EPT; ++j) any |= bal[j];
                if (!__syncthreads_or(any != 0)) continue;
                if (lane < EPT) {
                    unsigned mine = 0;
#pragma unroll
                    for (int j = 0; j < EPT; ++j)
                        if (lane == (unsigned)j) mine = __popc(bal[j]);
                    sm.jw[lane * NW + warp] = mine;
                }
                __syncthreads();
                if (warp == 0) {  // scan EPT*NW counts in (j, warp) order, CPL per lane
                    constexpr int CPL = EPT * NW / 32;
                    unsigned a[CPL], sum = 0;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) { a[q] = sm.jw[CPL * lane + q]; sum += a[q]; }
                    const unsigned incl = warp_incl_scan(sum);
                    unsigned run = incl - sum;
#pragma unroll
                    for (int q = 0; q < CPL; ++q) { sm.jw[CPL * lane + q] = run; run += a[q]; }
                    if (lane == 31) sm.tot = incl;
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < EPT; ++j)
                    if (bal[j] & (1u << lane)) out[written + sm.jw[j * NW + warp] + __popc(bal[j] & lanemask_lt())] = ids[j];
                written += sm.tot;
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) C->segcnt[np][blockIdx.x] = written;
        grid_sync(&C->bar, G);
        if (blockIdx.x == 0 && threadIdx.x == 0 && it < P.max_iters) {
            P.rec_ns[it] = (long long)(globaltimer() - t0);
            P.rec_size[it] = (long long)size;
            P.rec_cutoff[it] = cutoff;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->iters = it;
        C->overflow = it > P.max_iters;
    }
}

}  // namespace pushbench
}  // namespace hcb

using namespace hcb;
using namespace hcb::pushbench;

// G segments of capacity ceil(n/G) + 16 (shares are rounded to 16 elements)
static size_t seg_region_bytes(long long n) { return 4 * ((size_t)n + (size_t)MAXG * 32); }

static unsigned pb_grid() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pushbench_kernel, BLOCK, 0);
    long long g = (long long)per_sm * num_sms();
    if (g > MAXG) g = MAXG;
    return (unsigned)(g < 1 ? 1 : g);
}

extern "C" {

size_t hc_push_bench_workspace_bytes(int64_t n) {
    if (n < 0) n = 0;
    return align_up((size_t)n + 16, 256) + 2 * align_up(seg_region_bytes(n), 256) + align_up(sizeof(Ctrl), 256);
}

int hc_push_bench(int64_t n, int64_t batch, int variant, int64_t *d_rec_ns, int64_t *d_rec_size,
                  int64_t *d_rec_cutoff, int64_t max_iters, int64_t *h_iters, void *d_ws, size_t ws_bytes,
                  void *stream) {
    HC_REQUIRE(n >= 0 && n < 0x7fffffffLL && batch >= 1 && (variant == 0 || variant == 1) && max_iters >= 0,
               HC_ERR_INVALID, "push_bench: bad arguments");
    HC_REQUIRE(d_ws && ws_bytes >= hc_push_bench_workspace_bytes(n), HC_ERR_WORKSPACE,
               "push_bench: workspace too small");
    cudaStream_t st = as_stream(stream);
    if (h_iters) *h_iters = 0;
    if (n == 0) return HC_OK;
    const unsigned G = pb_grid();
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P;
    P.n = n;
    P.batch = batch;
    P.variant = variant;
    P.active = reinterpret_cast<unsigned char *>(ws);
    P.segcap = (n + G - 1) / G + 16;
    const size_t seg_bytes = align_up(seg_region_bytes(n), 256);
    P.seg[0] = reinterpret_cast<int *>(ws + align_up((size_t)n + 16, 256));
    P.seg[1] = reinterpret_cast<int *>(ws + align_up((size_t)n + 16, 256) + seg_bytes);
    P.ctrl = reinterpret_cast<Ctrl *>(ws + align_up((size_t)n + 16, 256) + 2 * seg_bytes);
    P.rec_ns = reinterpret_cast<long long *>(d_rec_ns);
    P.rec_size = reinterpret_cast<long long *>(d_rec_size);
    P.rec_cutoff = reinterpret_cast<long long *>(d_rec_cutoff);
    P.max_iters = max_iters;
    P.nblocks = G;
    HC_CUDA_TRY(cudaMemsetAsync(P.ctrl, 0, sizeof(Ctrl), st));
    void *args[] = {&P};
    HC_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)pushbench_kernel, dim3(G), dim3(BLOCK), args, 0, st));
    long long info[2];
    HC_CUDA_TRY(cudaMemcpyAsync(info, &P.ctrl->iters, sizeof info, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    if (h_iters) *h_iters = info[0];
    HC_REQUIRE(!info[1], HC_ERR_RECORDS, "push_bench: %lld iterations exceed the record buffer", info[0]);
    return HC_OK;
}

}  // extern "C"
