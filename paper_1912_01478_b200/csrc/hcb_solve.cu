// hcb_solve.cu -- device-resident IPGC solve (hc_solve).
//
// Replaces the reference's whole `color_graph` round loop
// (pkg/src/hybridcolor/driver.py:122-176) together with the round functions
// (coloring.py:113-176), the kernels (_kernels.pyx:29-149) and the worklist
// swap (worklist.py:77-91) by ONE cooperatively launched persistent kernel:
// every round is  assign -> grid barrier -> resolve -> grid barrier  with the
// hybrid mode decision, the worklist and the per-round records kept on the
// device, so there is no host round-trip per round.
//
// State encoding (one 32-bit word per node, X[u]):
//   X[u] == 0                 never assigned
//   X[u] == T (bit31 clear)   uncolored; T = tentative color of the current /
//                             last round (a loser keeps its stale T)
//   X[u] == C | FBIT          permanently colored with C
// Equivalence with the reference's (colors_read, colors_write, stamp) triple
// (SURVEY.md Appendix A):
//   * assign reads only committed colors: it ignores words without FBIT, which
//     is exactly "active neighbours read 0" (colors_read of a loser is reset by
//     the commit at coloring.py:140/174).
//   * resolve counts v<u with color(X[v]) == T[u].  The reference's extra test
//     stamp[v]==round (_kernels.pyx:113) is implied: a neighbour committed in an
//     earlier round has a color T[u] avoided (T[u] is the mex over committed
//     neighbour colors), and every uncolored node is active in every round
//     (data: worklist == {C==0}; topo: activity C==0).  Winners of the current
//     round set FBIT during resolve without changing the color bits, so
//     concurrent readers see the same color either way; losers keep T so they
//     still count for higher neighbours (test_coloring.py:84-91).
//   * winners commit C[u]=T[u] in resolve itself; no separate commit pass.
//
// Work distribution (IrGL-style nested parallelism):
// nodes are binned once by degree -- small (thread per node), mid (warp per
// node), hub (CTA per node).  The always-maintained worklist is kept per bin
// and double buffered; resolve pushes losers with warp-aggregated atomics.
// Topology-driven rounds sweep the static bin lists testing activity; data-
// driven rounds walk the dynamic lists.  Units are handed out dynamically:
// hubs first (CTA granularity), then mid nodes and small-node chunks (warp
// granularity), so the largest work items start first.
#include <algorithm>

#include "hcb_partition.cuh"

namespace hcb {
namespace solve {

constexpr int BLOCK = 256;
constexpr int NW = BLOCK / 32;
constexpr int SMALL_MAX = 16;            // deg <= SMALL_MAX : thread per node (64-bit mask mex)
constexpr int MID_WORDS = 64;            // warp bitmap words -> mid nodes up to 2046 neighbours
constexpr int MID_MAX = MID_WORDS * 32 - 2;
constexpr int HUB_WORDS = 512;           // CTA bitmap window: 16384 colors per pass
constexpr int SPL = 4;                   // small nodes per lane per warp unit
constexpr long long SMALL_UNIT = 32LL * SPL;
constexpr unsigned FBIT = 0x80000000u;
constexpr unsigned CMASK = 0x7fffffffu;

enum { BIN_SMALL = 0, BIN_MID = 1, BIN_HUB = 2, NBIN = 3 };

struct Ctrl {
    GridBarrier bar;
    int error;
    int pad0;
    unsigned long long nstat[NBIN];          // static bin sizes
    unsigned long long cnt[2][NBIN];         // worklist sizes per parity / bin
    unsigned long long conflicts[2];
    unsigned int hub_ctr[2][2];              // [phase][parity]
    unsigned int warp_ctr[2][2];
    long long rounds;
    long long rec_overflow;
};

struct Params {
    const long long *ro;
    const int *ci;
    long long n;
    unsigned *X;
    int *stat;          // static lists, bins contiguous
    int *dyn[2];        // dynamic lists per parity, same bin offsets as stat
    Ctrl *ctrl;
    hc_round_rec *rec;
    long long max_rec;
    long long *colors_out;
    int mode;
    long long thr;
    unsigned nblocks;
};

struct Smem {
    unsigned mid_bm[NW][MID_WORDS];
    unsigned hub_bm[HUB_WORDS];
    unsigned long long red;
    int hub_first;
    int unit;
    unsigned long long s_cnt[NBIN];
    int stop;
    int topo;
};

// ------------------------------------------------------------------ small
__device__ __forceinline__ unsigned assign_small(const Params &P, int u) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned long long mask = 0;
    for (long long k = b; k < e; k += 4) {
        int v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (k + j < e) ? P.ci[k + j] : -1;
        unsigned x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = v[j] >= 0 ? P.X[v[j]] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned c = x[j] & CMASK;
            if ((x[j] & FBIT) && c <= 64u) mask |= 1ull << (c - 1u);
        }
    }
    return (unsigned)__ffsll((long long)~mask);  // deg <= SMALL_MAX < 64: a zero bit exists
}

__device__ __forceinline__ unsigned resolve_small(const Params &P, int u, unsigned T) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned cnt = 0;
    for (long long k = b; k < e; k += 4) {
        int v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (k + j < e) ? P.ci[k + j] : 0x7fffffff;
        bool done = false;
        unsigned x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = v[j] < u ? P.X[v[j]] : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (v[j] < u) cnt += (x[j] & CMASK) == T;
            else done = true;
        }
        if (done) break;  // adjacency is sorted ascending (graph.py:193-197)
    }
    return cnt;
}

// ------------------------------------------------------------------ mid (warp)
__device__ __forceinline__ unsigned assign_mid(const Params &P, int u, unsigned *bm) {
    const unsigned lane = lane_id();
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;  // mex <= deg+1 (_kernels.pyx:49)
#pragma unroll
    for (int w = 0; w < MID_WORDS / 32; ++w) bm[lane + 32 * w] = 0u;
    __syncwarp();
    for (long long k = b + lane; k < e; k += 64) {
        const int v0 = P.ci[k];
        const int v1 = (k + 32 < e) ? P.ci[k + 32] : -1;
        const unsigned x0 = P.X[v0];
        const unsigned x1 = v1 >= 0 ? P.X[v1] : 0u;
        unsigned c = x0 & CMASK;
        if ((x0 & FBIT) && c <= lim) atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
        c = x1 & CMASK;
        if ((x1 & FBIT) && c <= lim) atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
    }
    __syncwarp();
    unsigned T = 0;
#pragma unroll
    for (int w = 0; w < MID_WORDS / 32; ++w) {
        const unsigned word = bm[lane + 32 * w];
        const unsigned bal = __ballot_sync(FULL, word != FULL);
        if (bal) {
            const int f = __ffs(bal) - 1;
            const unsigned fw = __shfl_sync(FULL, word, f);
            T = (unsigned)((w * 32 + f) * 32 + __ffs(~fw));
            break;
        }
    }
    __syncwarp();
    return T;
}

__device__ __forceinline__ unsigned resolve_mid(const Params &P, int u, unsigned T) {
    const unsigned lane = lane_id();
    const long long b = P.ro[u], e = P.ro[u + 1];
    unsigned cnt = 0;
    for (long long k0 = b; k0 < e; k0 += 32) {
        const long long k = k0 + lane;
        const int v = k < e ? P.ci[k] : 0x7fffffff;
        const bool lower = v < u;
        if (lower) cnt += (P.X[v] & CMASK) == T;
        if (__ballot_sync(FULL, !lower)) break;
    }
    return warp_sum(cnt);
}

// ------------------------------------------------------------------ hub (CTA)
__device__ unsigned assign_hub(const Params &P, int u, Smem &sm) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;
    for (unsigned w0 = 0;; w0 += HUB_WORDS * 32) {
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK) sm.hub_bm[i] = 0u;
        if (threadIdx.x == 0) sm.hub_first = 0x7fffffff;
        __syncthreads();
        const unsigned hi = min(lim, w0 + HUB_WORDS * 32);
        for (long long k = b + threadIdx.x; k < e; k += 2 * BLOCK) {
            const int v0 = P.ci[k];
            const int v1 = (k + BLOCK < e) ? P.ci[k + BLOCK] : -1;
            const unsigned x0 = P.X[v0];
            const unsigned x1 = v1 >= 0 ? P.X[v1] : 0u;
            unsigned c = x0 & CMASK;
            if ((x0 & FBIT) && c > w0 && c <= hi)
                atomicOr(&sm.hub_bm[(c - w0 - 1u) >> 5], 1u << ((c - w0 - 1u) & 31u));
            c = x1 & CMASK;
            if ((x1 & FBIT) && c > w0 && c <= hi)
                atomicOr(&sm.hub_bm[(c - w0 - 1u) >> 5], 1u << ((c - w0 - 1u) & 31u));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK)
            if (sm.hub_bm[i] != FULL) { atomicMin(&sm.hub_first, i); break; }
        __syncthreads();
        const int f = sm.hub_first;
        if (f != 0x7fffffff) {
            const unsigned T = w0 + (unsigned)f * 32u + (unsigned)__ffs(~sm.hub_bm[f]);
            __syncthreads();
            return T;
        }
        __syncthreads();
    }
}

__device__ unsigned resolve_hub(const Params &P, int u, unsigned T, Smem &sm) {
    const long long b = P.ro[u], e = P.ro[u + 1];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    if (threadIdx.x == 0) sm.red = 0;
    __syncthreads();
    unsigned cnt = 0;
    for (long long k0 = b + (long long)warp * 32; k0 < e; k0 += (long long)BLOCK) {
        const long long k = k0 + lane;
        const int v = k < e ? P.ci[k] : 0x7fffffff;
        const bool lower = v < u;
        if (lower) cnt += (P.X[v] & CMASK) == T;
        if (__ballot_sync(FULL, !lower)) break;  // later chunks are all >= u
    }
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&sm.red, (unsigned long long)cnt);
    __syncthreads();
    const unsigned total = (unsigned)sm.red;
    __syncthreads();
    return total;
}

// ------------------------------------------------------------------ pushes
__device__ __forceinline__ void push_one(const Params &P, int *list, int bin, int np, int u) {
    const unsigned long long pos = atomicAdd(&P.ctrl->cnt[np][bin], 1ull);
    list[pos] = u;
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(BLOCK, 4) solve_kernel(Params P) {
    __shared__ Smem sm;
    Ctrl *C = P.ctrl;
    const unsigned lane = lane_id();
    const unsigned warp = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long gthreads = (long long)P.nblocks * BLOCK;

    for (long long u = gtid; u < P.n; u += gthreads) P.X[u] = 0u;
    const unsigned long long nst[NBIN] = {C->nstat[0], C->nstat[1], C->nstat[2]};
    const unsigned long long off[NBIN] = {0, nst[0], nst[0] + nst[1]};
    const bool ident_small = nst[0] == (unsigned long long)P.n;  // all nodes small: sweep ids
    grid_sync(&C->bar, P.nblocks);

    unsigned long long t_start = 0;
    long long wl_in_prev = 0;
    int topo_prev = 0;
    unsigned long long my_conf = 0;
    long long t = 1;
    for (;; ++t) {
        const int p = (int)(t & 1), np = p ^ 1;
        if (threadIdx.x < NBIN) sm.s_cnt[threadIdx.x] = ld_relaxed_u64(&C->cnt[p][threadIdx.x]);
        __syncthreads();
        const unsigned long long sz[NBIN] = {sm.s_cnt[0], sm.s_cnt[1], sm.s_cnt[2]};
        const unsigned long long s = sz[0] + sz[1] + sz[2];
        const bool topo =
            P.mode == HC_MODE_TOPO || (P.mode == HC_MODE_HYBRID && (long long)s > P.thr);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const unsigned long long now = globaltimer();
            if (t > 1) {  // finish the record of round t-1 (driver.py:159-168)
                const int q = (int)((t - 1) & 1);
                if (t - 1 <= P.max_rec) {
                    hc_round_rec r;
                    r.round = t - 1;
                    r.topo = topo_prev;
                    r.wl_in = wl_in_prev;
                    r.wl_out = (long long)s;
                    r.conflicts = (long long)C->conflicts[q];
                    r.ns = (long long)(now - t_start);
                    P.rec[t - 2] = r;
                }
                C->conflicts[q] = 0;
                for (int bb = 0; bb < NBIN; ++bb) C->cnt[q][bb] = 0;
                C->hub_ctr[0][q] = C->hub_ctr[1][q] = 0;
                C->warp_ctr[0][q] = C->warp_ctr[1][q] = 0;
            }
            t_start = now;
            wl_in_prev = (long long)s;
            topo_prev = topo;
        }
        if (s == 0) break;  // worklist drained (driver.py:145)

        // lists of this round
        const int *lst = (t == 1 || topo) ? P.stat : P.dyn[p];
        const unsigned long long nh = topo ? nst[BIN_HUB] : sz[BIN_HUB];
        const unsigned long long nm = topo ? nst[BIN_MID] : sz[BIN_MID];
        const unsigned long long ns = topo ? nst[BIN_SMALL] : sz[BIN_SMALL];
        const bool ident = topo && ident_small;
        const unsigned long long mid_units = nm;
        const unsigned long long small_units = (ns + SMALL_UNIT - 1) / SMALL_UNIT;
        int *nxt = P.dyn[np];

        for (int phase = 0; phase < 2; ++phase) {
            // ---- hubs: one CTA per node
            for (;;) {
                if (threadIdx.x == 0) sm.unit = (int)atomicAdd(&C->hub_ctr[phase][p], 1u);
                __syncthreads();
                const unsigned long long unit = (unsigned)sm.unit;
                __syncthreads();
                if (unit >= nh) break;
                const int u = lst[off[BIN_HUB] + unit];
                const unsigned xu = P.X[u];
                if (topo && (xu & FBIT)) continue;  // topology sweep: inactive (_kernels.pyx:76)
                if (phase == 0) {
                    const unsigned T = assign_hub(P, u, sm);
                    if (threadIdx.x == 0) P.X[u] = T;
                } else {
                    const unsigned k = resolve_hub(P, u, xu, sm);
                    if (threadIdx.x == 0) {
                        my_conf += k;
                        if (k) push_one(P, nxt + off[BIN_HUB], BIN_HUB, np, u);
                        else P.X[u] = xu | FBIT;
                    }
                }
            }
            // ---- mid nodes (warp per node) then small chunks (thread per node)
            unsigned long long unit;
            if (lane == 0) unit = atomicAdd(&C->warp_ctr[phase][p], 1u);
            unit = __shfl_sync(FULL, unit, 0);
            while (unit < mid_units + small_units) {
                unsigned long long next_unit;
                if (lane == 0) next_unit = atomicAdd(&C->warp_ctr[phase][p], 1u);
                if (unit < mid_units) {
                    const int u = lst[off[BIN_MID] + unit];
                    const unsigned xu = P.X[u];
                    if (!(topo && (xu & FBIT))) {
                        if (phase == 0) {
                            const unsigned T = assign_mid(P, u, sm.mid_bm[warp]);
                            if (lane == 0) P.X[u] = T;
                        } else {
                            const unsigned k = resolve_mid(P, u, xu);
                            if (lane == 0) {
                                my_conf += k;
                                if (k) push_one(P, nxt + off[BIN_MID], BIN_MID, np, u);
                                else P.X[u] = xu | FBIT;
                            }
                        }
                    }
                } else {
                    const unsigned long long base = (unit - mid_units) * SMALL_UNIT;
#pragma unroll 1
                    for (int j = 0; j < SPL; ++j) {
                        const unsigned long long idx = base + (unsigned long long)j * 32 + lane;
                        int u = -1;
                        unsigned xu = 0;
                        if (idx < ns) {
                            u = ident ? (int)idx : lst[off[BIN_SMALL] + idx];
                            xu = P.X[u];
                            if (topo && (xu & FBIT)) u = -1;
                        }
                        bool lost = false;
                        if (u >= 0) {
                            if (phase == 0) {
                                P.X[u] = assign_small(P, u);
                            } else {
                                const unsigned k = resolve_small(P, u, xu);
                                my_conf += k;
                                lost = k != 0;
                                if (!lost) P.X[u] = xu | FBIT;
                            }
                        }
                        if (phase == 1) {  // warp-aggregated push
                            const unsigned bal = __ballot_sync(FULL, lost);
                            if (bal) {
                                unsigned long long basepos = 0;
                                if (lane == 0)
                                    basepos = atomicAdd(&C->cnt[np][BIN_SMALL], (unsigned long long)__popc(bal));
                                basepos = __shfl_sync(FULL, basepos, 0);
                                if (lost)
                                    nxt[off[BIN_SMALL] + basepos + __popc(bal & lanemask_lt())] = u;
                            }
                        }
                    }
                }
                unit = __shfl_sync(FULL, next_unit, 0);
            }
            if (phase == 0) grid_sync(&C->bar, P.nblocks);
        }
        // conflicts of this round: block reduce then one atomic per CTA
        {
            unsigned long long v = warp_sum(my_conf);
            my_conf = 0;
            if (threadIdx.x == 0) sm.red = 0;
            __syncthreads();
            if (lane == 0 && v) atomicAdd(&sm.red, v);
            __syncthreads();
            if (threadIdx.x == 0 && sm.red) atomicAdd(&C->conflicts[p], sm.red);
        }
        grid_sync(&C->bar, P.nblocks);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->rounds = t - 1;
        if (t - 1 > P.max_rec) C->rec_overflow = 1;
    }
    for (long long u = gtid; u < P.n; u += gthreads) P.colors_out[u] = (long long)(P.X[u] & CMASK);
}

// degree classifier for the static bins
struct DegreeBin {
    const long long *ro;
    __device__ int operator()(long long i) const {
        const long long d = ro[i + 1] - ro[i];
        return d <= SMALL_MAX ? BIN_SMALL : (d <= MID_MAX ? BIN_MID : BIN_HUB);
    }
};
struct EmitI32 {
    __device__ int operator()(long long i) const { return (int)i; }
};

__global__ void copy_totals_kernel(const unsigned long long *totals, Ctrl *c) {
    if (threadIdx.x < NBIN) {
        c->nstat[threadIdx.x] = totals[threadIdx.x];
        c->cnt[1][threadIdx.x] = totals[threadIdx.x];  // W_1 = all nodes (worklist.py:37-39)
    }
}

struct Layout {
    size_t x, stat, dyn0, dyn1, ctrl, part, total;
};

static Layout layout(long long n) {
    Layout L;
    size_t o = 0;
    L.x = o; o = align_up(o + 4 * (size_t)n, 256);
    L.stat = o; o = align_up(o + 4 * (size_t)n, 256);
    L.dyn0 = o; o = align_up(o + 4 * (size_t)n, 256);
    L.dyn1 = o; o = align_up(o + 4 * (size_t)n, 256);
    L.ctrl = o; o = align_up(o + sizeof(Ctrl), 256);
    L.part = o; o = align_up(o + part_scratch_bytes(NBIN, n), 256);
    L.total = o;
    return L;
}

static int occupancy() {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel, BLOCK, 0) != cudaSuccess)
        return 0;
    return per_sm;
}

}  // namespace solve
}  // namespace hcb

using namespace hcb;
using namespace hcb::solve;

extern "C" {

int hc_device_info(int *h_num_sms, int *h_ctas_per_sm) {
    if (h_num_sms) *h_num_sms = num_sms();
    if (h_ctas_per_sm) *h_ctas_per_sm = occupancy();
    return HC_OK;
}

size_t hc_solve_workspace_bytes(int64_t num_nodes, int64_t num_edges) {
    (void)num_edges;
    return layout(num_nodes < 0 ? 0 : num_nodes).total;
}

int hc_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
             int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
             int64_t max_rec, int64_t *h_rounds, void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(num_nodes >= 0 && num_nodes < 0x7fffffffLL, HC_ERR_INVALID,
               "hc_solve: num_nodes %lld out of range", (long long)num_nodes);
    HC_REQUIRE(mode >= HC_MODE_DATA && mode <= HC_MODE_HYBRID, HC_ERR_INVALID,
               "hc_solve: mode %d invalid", mode);
    HC_REQUIRE(max_rec >= 0, HC_ERR_INVALID, "hc_solve: max_rec < 0");
    cudaStream_t st = as_stream(stream);
    if (h_rounds) *h_rounds = 0;
    if (num_nodes == 0) return HC_OK;  // empty graph: 0 rounds (test_driver.py:88-93)
    HC_REQUIRE(d_row_offsets && d_colors && (num_edges == 0 || d_col_indices), HC_ERR_INVALID,
               "hc_solve: null pointer");
    const Layout L = layout(num_nodes);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_solve: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P;
    P.ro = reinterpret_cast<const long long *>(d_row_offsets);
    P.ci = d_col_indices;
    P.n = num_nodes;
    P.X = reinterpret_cast<unsigned *>(ws + L.x);
    P.stat = reinterpret_cast<int *>(ws + L.stat);
    P.dyn[0] = reinterpret_cast<int *>(ws + L.dyn0);
    P.dyn[1] = reinterpret_cast<int *>(ws + L.dyn1);
    P.ctrl = reinterpret_cast<Ctrl *>(ws + L.ctrl);
    P.rec = d_rec;
    P.max_rec = d_rec ? max_rec : 0;
    P.colors_out = reinterpret_cast<long long *>(d_colors);
    P.mode = mode;
    P.thr = thr_count;

    HC_CUDA_TRY(cudaMemsetAsync(P.ctrl, 0, sizeof(Ctrl), st));
    unsigned long long *totals = nullptr;
    int rc = ordered_partition<NBIN>(num_nodes, DegreeBin{P.ro}, EmitI32{}, P.stat, ws + L.part,
                                     &totals, st);
    if (rc != HC_OK) return rc;
    copy_totals_kernel<<<1, 32, 0, st>>>(totals, P.ctrl);
    HC_CHECK_LAUNCH();

    const int per_sm = occupancy();
    const int sms = num_sms();
    HC_REQUIRE(per_sm > 0 && sms > 0, HC_ERR_CUDA, "hc_solve: occupancy query failed");
    P.nblocks = (unsigned)(per_sm * sms);
    void *args[] = {&P};
    HC_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)solve_kernel, dim3(P.nblocks), dim3(BLOCK),
                                            args, 0, st));
    long long info[2];
    HC_CUDA_TRY(cudaMemcpyAsync(info, &P.ctrl->rounds, sizeof info, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    if (h_rounds) *h_rounds = info[0];
    HC_REQUIRE(!info[1], HC_ERR_RECORDS, "hc_solve: %lld rounds exceed the %lld-record buffer",
               info[0], (long long)max_rec);
    return HC_OK;
}

}  // extern "C"
