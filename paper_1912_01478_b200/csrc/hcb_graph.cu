// hcb_graph.cu -- device graph construction, synthetic generators and
// verification.
//
//   hc_build_csr   <- build_csr, pkg/src/hybridcolor/graph.py:184-201
//   hc_gen_*       <- SURVEY.md Appendix C (bit-identical to oracle/ipgc_oracle.c)
//   hc_verify      <- verify_coloring, driver.py:188-204
//   hc_colors_used <- colors_used, driver.py:179-185
//
// CSR build = counting sort by source + per-row sort/dedupe instead of the
// reference's global np.unique over src*n+dst (same result: rows ascending,
// duplicates and loops dropped):
//   1. degree count (both directions, loops dropped)     atomics, 1 pass
//   2. exclusive scan -> row starts                        3-kernel scan
//   3. scatter both directions into the row slots          atomic cursors
//   4. per-row sort + dedupe, binned by row length:
//        <= 64      warp per row, register bitonic network
//        <= 8192    CTA per row, shared-memory bitonic sort
//        larger     CTA per row, node-id bitmap (marks dedupe for free and
//                   the ordered bitmap scan emits the row sorted)
//   5. exclusive scan of unique counts -> row_offsets; 6. compact into int32.
#include <algorithm>

#include "hcb_partition.cuh"

namespace hcb {
namespace graph {

constexpr int BLOCK = 256;

__host__ __device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    unsigned long long z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long ghash(unsigned long long seed, unsigned long long k,
                                                    unsigned long long l) {
    return splitmix64((seed << 40) + (k << 6) + l);
}

constexpr unsigned long long RMAT_TA = 2448131359ULL;
constexpr unsigned long long RMAT_TB = 3264175145ULL;
constexpr unsigned long long RMAT_TC = 4080218931ULL;

inline unsigned grid_cap(long long items, int per_block) {
    long long g = (items + per_block - 1) / per_block;
    const long long cap = (long long)num_sms() * 64;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

__global__ void gen_grid_kernel(long long rows, long long cols, long long m, longlong2 *edges) {
    const long long per_row = 2 * cols - 1;
    const long long full = (rows - 1) * per_row;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        long long u, v;
        if (k < full) {
            const long long i = k / per_row, r = k - i * per_row;
            const long long j = r >> 1;
            u = i * cols + j;
            v = (r & 1) ? u + 1 : u + cols;  // conftest.py:37-40: down then right
        } else {
            const long long j = k - full;
            u = (rows - 1) * cols + j;
            v = u + 1;
        }
        edges[k] = make_longlong2(u, v);
    }
}

__global__ void gen_er_kernel(unsigned long long n, long long m, unsigned long long seed,
                              longlong2 *edges) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        edges[k] = make_longlong2((long long)(ghash(seed, k, 0) % n), (long long)(ghash(seed, k, 1) % n));
    }
}

__global__ void gen_rmat_kernel(int scale, long long m, unsigned long long seed, longlong2 *edges) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        long long s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            const unsigned long long r = ghash(seed, k, l) >> 32;
            const long long sb = r >= RMAT_TB;
            const long long db = (r >= RMAT_TA && r < RMAT_TB) || r >= RMAT_TC;
            s |= sb << l;
            d |= db << l;
        }
        edges[k] = make_longlong2(s, d);
    }
}

// ------------------------------------------------------------- scan u32->u64
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr long long SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) tile_sum_kernel(const unsigned *in, long long count,
                                                                unsigned long long *tile_sums) {
    __shared__ unsigned long long s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * SCAN_TILE;
    unsigned long long local = 0;
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const long long i = base + (long long)j * SCAN_THREADS + threadIdx.x;
        if (i < count) local += in[i];
    }
    local = warp_sum(local);
    if (lane_id() == 0 && local) atomicAdd(&s, local);
    __syncthreads();
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = s;
}

__global__ void __launch_bounds__(SCAN_THREADS) tile_scan_kernel(const unsigned *in, long long count,
                                                                 const unsigned long long *tile_offs,
                                                                 unsigned long long *out) {
    __shared__ unsigned long long s_warp[SCAN_THREADS / 32];
    const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    unsigned v[SCAN_ITEMS];
    unsigned long long local = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        v[j] = base + j < count ? in[base + j] : 0u;
        local += v[j];
    }
    unsigned long long incl = warp_incl_scan(local);
    const unsigned warp = threadIdx.x >> 5;
    if (lane_id() == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long x = lane_id() < SCAN_THREADS / 32 ? s_warp[lane_id()] : 0;
        unsigned long long xi = warp_incl_scan(x);
        if (lane_id() < SCAN_THREADS / 32) s_warp[lane_id()] = xi - x;
    }
    __syncthreads();
    unsigned long long run = tile_offs[blockIdx.x] + s_warp[warp] + incl - local;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        if (base + j < count) out[base + j] = run;
        run += v[j];
    }
    if (base < count && count <= base + SCAN_ITEMS) out[count] = run;  // total (owner of the last item)
}

inline size_t scan_scratch_bytes(long long count) {
    return align_up(sizeof(unsigned long long) * (size_t)((count + SCAN_TILE - 1) / SCAN_TILE + 1), 256) +
           256;
}

// out[0..count] (count+1 values): exclusive scan, out[count] = total
static int exclusive_scan(const unsigned *in, long long count, unsigned long long *out, void *scratch,
                          cudaStream_t st) {
    if (count == 0) {
        HC_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(unsigned long long), st));
        return HC_OK;
    }
    const long long tiles = (count + SCAN_TILE - 1) / SCAN_TILE;
    unsigned long long *tile_sums = reinterpret_cast<unsigned long long *>(scratch);
    unsigned long long *dummy = reinterpret_cast<unsigned long long *>(
        reinterpret_cast<char *>(scratch) + align_up(sizeof(unsigned long long) * (size_t)(tiles + 1), 256));
    tile_sum_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, count, tile_sums);
    HC_CHECK_LAUNCH();
    part_scan_kernel<<<1, PART_SCAN_THREADS, 0, st>>>(tile_sums, tiles, 1, tiles, dummy);
    HC_CHECK_LAUNCH();
    tile_scan_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, count, tile_sums, out);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

// ------------------------------------------------------------- csr build
// Rows [lo, hi) of the CSR (the whole graph: lo = 0, hi = n; a multi-GPU
// shard: the rank's owned range, with global column ids).  Row r = node lo+r.
__global__ void degree_kernel(const longlong2 *edges, long long m, long long n, long long lo, long long hi,
                              unsigned *deg, unsigned *status) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        const longlong2 e = edges[k];
        if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n) {
            atomicOr(status, 1u);
            continue;
        }
        if (e.x == e.y) continue;  // graph.py:192
        if (e.x >= lo && e.x < hi) atomicAdd(&deg[e.x - lo], 1u);
        if (e.y >= lo && e.y < hi) atomicAdd(&deg[e.y - lo], 1u);
    }
}

__global__ void scatter_kernel(const longlong2 *edges, long long m, long long n, long long lo, long long hi,
                               unsigned long long *cur, int *tmp) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        const longlong2 e = edges[k];
        if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n || e.x == e.y) continue;
        // graph.py:191 both directions
        if (e.x >= lo && e.x < hi) tmp[atomicAdd(&cur[e.x - lo], 1ull)] = (int)e.y;
        if (e.y >= lo && e.y < hi) tmp[atomicAdd(&cur[e.y - lo], 1ull)] = (int)e.x;
    }
}

// raw half-edge count per node (loops dropped, duplicates counted): the
// multi-GPU partition is cut on its prefix before any rank builds its shard
__global__ void raw_degree_kernel(const longlong2 *edges, long long m, long long n,
                                  unsigned long long *deg) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        const longlong2 e = edges[k];
        if (e.x < 0 || e.x >= n || e.y < 0 || e.y >= n || e.x == e.y) continue;
        atomicAdd(&deg[e.x], 1ull);
        atomicAdd(&deg[e.y], 1ull);
    }
}

// multi-GPU verify of a shard: edges u<v of the owned rows with equal colors
// or an uncolored u, colors indexed by global id (driver.py:188-204)
__global__ void verify_rows_kernel(const long long *ro, const int *ci, long long lo, long long nrows,
                                   const long long *colors, unsigned long long *acc) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long bad = 0;
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nwarps) {
        const long long u = lo + r, cu = colors[u];
        for (long long k = ro[r] + lane; k < ro[r + 1]; k += 32) {
            const long long v = ci[k];
            if (u < v && (cu == colors[v] || cu == 0)) ++bad;
        }
    }
    bad = warp_sum(bad);
    if (lane == 0 && bad) atomicAdd(acc, bad);
}

constexpr int SMALL_ROW = 64;
constexpr int MID_ROW = 8192;
constexpr int MID_THREADS = 512;

// warp per row, rows of <= 64 entries: bitonic network in registers
__global__ void sort_small_rows_kernel(const unsigned long long *off, long long n, int *tmp,
                                       unsigned *uniq) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const unsigned long long b = off[u], e = off[u + 1];
        const unsigned d = (unsigned)(e - b);
        if (d > SMALL_ROW) continue;
        if (d <= 1) {
            if (lane == 0) uniq[u] = d;
            continue;
        }
        int a0 = lane < d ? tmp[b + lane] : 0x7fffffff;
        int a1 = lane + 32 < d ? tmp[b + lane + 32] : 0x7fffffff;
        // bitonic sort of 64 keys, key index i = lane + 32*r
#pragma unroll
        for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                if (j == 32) {
                    // partner of (lane, r=0) is (lane, r=1); ascending iff (i & k)==0, i<64 -> k=64: asc
                    const int lo = min(a0, a1), hi = max(a0, a1);
                    a0 = lo;
                    a1 = hi;
                } else {
                    const int p0 = __shfl_xor_sync(FULL, a0, j);
                    const int p1 = __shfl_xor_sync(FULL, a1, j);
                    const unsigned i0 = lane, i1 = lane + 32;
                    const bool up0 = (i0 & k) == 0, up1 = (i1 & k) == 0;
                    const bool low0 = (i0 & j) == 0, low1 = (i1 & j) == 0;
                    a0 = (low0 == up0) ? min(a0, p0) : max(a0, p0);
                    a1 = (low1 == up1) ? min(a1, p1) : max(a1, p1);
                }
            }
        }
        // dedupe (sorted order: a0 of lanes 0..31, then a1 of lanes 0..31)
        const int prev0 = __shfl_up_sync(FULL, a0, 1);
        int prev1 = __shfl_up_sync(FULL, a1, 1);
        const int last0 = __shfl_sync(FULL, a0, 31);
        if (lane == 0) prev1 = last0;
        const bool f0 = a0 != 0x7fffffff && (lane == 0 || a0 != prev0);
        const bool f1 = a1 != 0x7fffffff && a1 != prev1;
        const unsigned b0 = __ballot_sync(FULL, f0), b1 = __ballot_sync(FULL, f1);
        const unsigned c0 = __popc(b0);
        if (f0) tmp[b + __popc(b0 & lanemask_lt())] = a0;
        if (f1) tmp[b + c0 + __popc(b1 & lanemask_lt())] = a1;
        if (lane == 0) uniq[u] = c0 + __popc(b1);
    }
}

// CTA per row, 64 < rows <= MID_ROW: shared-memory bitonic sort + ordered dedupe
__global__ void __launch_bounds__(MID_THREADS) sort_mid_rows_kernel(const unsigned long long *off,
                                                                    const int *rows, long long nrows,
                                                                    int *tmp, unsigned *uniq) {
    __shared__ int s[MID_ROW];
    __shared__ unsigned s_warp[MID_THREADS / 32];
    for (long long r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int u = rows[r];
        const unsigned long long b = off[u];
        const unsigned d = (unsigned)(off[u + 1] - b);
        unsigned P = 128;
        while (P < d) P <<= 1;
        for (unsigned i = threadIdx.x; i < P; i += MID_THREADS) s[i] = i < d ? tmp[b + i] : 0x7fffffff;
        __syncthreads();
        for (unsigned k = 2; k <= P; k <<= 1) {
            for (unsigned j = k >> 1; j > 0; j >>= 1) {
                for (unsigned i = threadIdx.x; i < P; i += MID_THREADS) {
                    const unsigned l = i ^ j;
                    if (l > i) {
                        const int x = s[i], y = s[l];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            s[i] = y;
                            s[l] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // ordered dedupe: each thread owns a contiguous chunk of P/MID_THREADS
        const unsigned per = (P + MID_THREADS - 1) / MID_THREADS;
        const unsigned lo = min(P, per * threadIdx.x), hi = min(P, lo + per);
        unsigned cnt = 0;
        for (unsigned i = lo; i < hi; ++i)
            cnt += s[i] != 0x7fffffff && (i == 0 || s[i] != s[i - 1]);
        const unsigned incl = warp_incl_scan(cnt);
        const unsigned warp = threadIdx.x >> 5;
        if (lane_id() == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned x = lane_id() < MID_THREADS / 32 ? s_warp[lane_id()] : 0;
            const unsigned xi = warp_incl_scan(x);
            if (lane_id() < MID_THREADS / 32) s_warp[lane_id()] = xi - x;
            if (lane_id() == MID_THREADS / 32 - 1) uniq[u] = xi;
        }
        __syncthreads();
        unsigned pos = s_warp[warp] + incl - cnt;
        for (unsigned i = lo; i < hi; ++i)
            if (s[i] != 0x7fffffff && (i == 0 || s[i] != s[i - 1])) tmp[b + pos++] = s[i];
        __syncthreads();
    }
}

// CTA per row, rows > MID_ROW: per-CTA node bitmap (n bits) plus a summary
// bitmap (one bit per bitmap word) -> sorted unique.  The emit pass walks the
// summary only, so a row costs O(n/1024 + its entries), not O(n/32): RMAT-26
// (67 M nodes, ~10 K rows above MID_ROW) scanned 8 MB of bitmap per row
// (868 ms of a 1.3 s build).
__global__ void __launch_bounds__(BLOCK) sort_big_rows_kernel(const unsigned long long *off,
                                                              const int *rows, long long nrows,
                                                              long long n, int *tmp, unsigned *uniq,
                                                              unsigned *bitmaps, unsigned *summaries) {
    __shared__ unsigned s_warp[BLOCK / 32];
    __shared__ unsigned long long s_base;
    const long long words = (n + 31) / 32, swords = (words + 31) / 32;
    unsigned *bm = bitmaps + (long long)blockIdx.x * words;
    unsigned *sm = summaries + (long long)blockIdx.x * swords;
    for (long long r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int u = rows[r];
        const unsigned long long b = off[u], e = off[u + 1];
        for (unsigned long long k = b + threadIdx.x; k < e; k += BLOCK) {
            const int v = tmp[k];
            const int w = v >> 5;
            // the setter that finds the word empty marks it in the summary
            if (atomicOr(&bm[w], 1u << (v & 31)) == 0u) atomicOr(&sm[w >> 5], 1u << (w & 31));
        }
        __syncthreads();  // bitmaps complete (block-local atomics at L2, ordered by bar)
        __threadfence_block();
        if (threadIdx.x == 0) s_base = 0;
        __syncthreads();
        for (long long s0 = 0; s0 < swords; s0 += BLOCK) {
            const long long sw = s0 + threadIdx.x;
            const unsigned sword = sw < swords ? __ldcg(&sm[sw]) : 0u;
            unsigned c = 0;
            for (unsigned q = sword; q; q &= q - 1u) c += __popc(__ldcg(&bm[sw * 32 + (__ffs(q) - 1)]));
            const unsigned incl = warp_incl_scan(c);
            const unsigned warp = threadIdx.x >> 5;
            if (lane_id() == 31) s_warp[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                const unsigned x = lane_id() < BLOCK / 32 ? s_warp[lane_id()] : 0;
                const unsigned xi = warp_incl_scan(x);
                if (lane_id() < BLOCK / 32) s_warp[lane_id()] = xi - x;
            }
            __syncthreads();
            unsigned long long pos = b + s_base + s_warp[warp] + incl - c;
            if (sword) {
                sm[sw] = 0u;  // leave both bitmaps clean for the next row
                for (unsigned q = sword; q; q &= q - 1u) {
                    const long long w = sw * 32 + (__ffs(q) - 1);
                    unsigned word = __ldcg(&bm[w]);
                    bm[w] = 0u;
                    while (word) {
                        const int bit = __ffs(word) - 1;
                        word &= word - 1;
                        tmp[pos++] = (int)(w * 32 + bit);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == BLOCK - 1) s_base += s_warp[warp] + incl;
            __syncthreads();
        }
        if (threadIdx.x == 0) uniq[u] = (unsigned)s_base;
        __syncthreads();
    }
}

struct RowBin {
    const unsigned long long *off;
    __device__ int operator()(long long u) const {
        const unsigned long long d = off[u + 1] - off[u];
        return d <= SMALL_ROW ? -1 : (d <= MID_ROW ? 0 : 1);
    }
};
struct EmitRow {
    __device__ int operator()(long long u) const { return (int)u; }
};

__global__ void compact_kernel(const unsigned long long *off, const unsigned long long *ro,
                               const int *tmp, long long n, int *ci) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const unsigned long long src = off[u], dst = ro[u], len = ro[u + 1] - ro[u];
        for (unsigned long long k = lane; k < len; k += 32) ci[dst + k] = tmp[src + k];
    }
}

// ------------------------------------------------------------- verify etc.
__global__ void verify_kernel(const long long *ro, const int *ci, long long n, const long long *colors,
                              unsigned long long *acc) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long bad = 0;
    for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const long long cu = colors[u];
        for (long long k = ro[u] + lane; k < ro[u + 1]; k += 32) {
            const long long v = ci[k];
            if (u < v && (cu == colors[v] || cu == 0)) ++bad;  // driver.py:202-204
        }
    }
    bad = warp_sum(bad);
    if (lane == 0 && bad) atomicAdd(acc, bad);
}

__global__ void colors_used_kernel(const long long *colors, long long n, unsigned long long *acc) {
    // acc[0] = max color, acc[1] = count of entries < 1
    unsigned long long mx = 0, bad = 0;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n;
         u += (long long)gridDim.x * blockDim.x) {
        const long long c = colors[u];
        if (c < 1) ++bad;
        else if ((unsigned long long)c > mx) mx = (unsigned long long)c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
    bad = warp_sum(bad);
    if (lane_id() == 0) {
        if (mx) atomicMax(&acc[0], mx);
        if (bad) atomicAdd(&acc[1], bad);
    }
}

__global__ void narrow_kernel(const long long *in, int *out, long long count) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (int)in[i];
}


// ------------------------------------------------------ lower-id-first rows
// The fused solver's resolve stops scanning a row at its first neighbour >= u
// (hcb_solve.cu), so it needs every row's lower-id neighbours to form a prefix
// of the row.  build_csr output (graph.py:193-197: sorted ascending) has that
// property; an arbitrary caller CSR may not.  The reference resolve scans the
// whole row (_kernels.pyx:106-113) and every solve output is a function of the
// row *sets* (mex, the v<u conflict count), so a stable partition of each row
// into (v < u) then (v >= u) changes nothing but the scan order.
__global__ void lower_first_check_kernel(const long long *ro, const int *ci, long long n,
                                         unsigned long long *acc) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long bad = 0;
    for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        bool seen_high = false, violates = false;
        for (long long k0 = ro[u]; k0 < ro[u + 1] && !violates; k0 += 32) {
            const long long k = k0 + lane;
            const bool in = k < ro[u + 1];
            const long long v = in ? ci[k] : 0;
            const unsigned high = __ballot_sync(FULL, in && v >= u);
            const unsigned low = __ballot_sync(FULL, in && v < u);
            if (seen_high && low) violates = true;
            // a low after the first high inside this chunk
            if (high && (low >> (__ffs(high) - 1)) != 0u) violates = true;
            seen_high |= high != 0u;
        }
        bad += (violates && lane == 0);
    }
    bad = warp_sum(bad);
    if (lane == 0 && bad) atomicAdd(acc, bad);
}

__global__ void lower_first_partition_kernel(const long long *ro, const int *in, int *out, long long n) {
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nwarps) {
        const long long b = ro[u], e = ro[u + 1];
        long long w = b;
        for (int pass = 0; pass < 2; ++pass) {
            for (long long k0 = b; k0 < e; k0 += 32) {
                const long long k = k0 + lane;
                const int v = k < e ? in[k] : 0;
                const bool take = k < e && ((pass == 0) == ((long long)v < u));
                const unsigned m = __ballot_sync(FULL, take);
                if (take) out[w + __popc(m & ((1u << lane) - 1u))] = v;
                w += __popc(m);
            }
        }
    }
}

struct CsrLayout {
    size_t deg, off, cur, tmp, uniq, ro_u, rows, status, bitmaps, summaries, scan, part, total;
    int big_ctas;
};

// n = the graph's node count (bitmap width), rows = rows built, dir = the
// directed (pre-dedupe) entries of those rows (2m for the whole graph)
static CsrLayout csr_layout(long long n, long long rows, long long dir) {
    CsrLayout L;
    size_t o = 0;
    L.big_ctas = num_sms() > 0 ? num_sms() : 148;
    L.deg = o; o = align_up(o + 4 * (size_t)(rows + 1), 256);
    L.off = o; o = align_up(o + 8 * (size_t)(rows + 1), 256);
    L.cur = o; o = align_up(o + 8 * (size_t)(rows + 1), 256);
    L.tmp = o; o = align_up(o + 4 * (size_t)(dir + 1), 256);
    L.uniq = o; o = align_up(o + 4 * (size_t)(rows + 1), 256);
    L.ro_u = o; o = align_up(o + 8 * (size_t)(rows + 1), 256);
    L.rows = o; o = align_up(o + 4 * (size_t)(rows + 1), 256);
    L.status = o; o = align_up(o + 256, 256);
    L.bitmaps = o; o = align_up(o + 4 * (size_t)((n + 31) / 32) * (size_t)L.big_ctas, 256);
    L.summaries = o; o = align_up(o + 4 * (size_t)((n + 1023) / 1024) * (size_t)L.big_ctas, 256);
    L.scan = o; o = align_up(o + scan_scratch_bytes(rows + 1), 256);
    L.part = o; o = align_up(o + part_scratch_bytes(2, rows), 256);
    L.total = o;
    return L;
}

}  // namespace graph
}  // namespace hcb

using namespace hcb;
using namespace hcb::graph;

extern "C" {

int hc_gen_grid(int64_t rows, int64_t cols, int64_t *d_edges, void *stream) {
    HC_REQUIRE(rows >= 0 && cols >= 0, HC_ERR_INVALID, "gen_grid: negative size");
    if (rows == 0 || cols == 0) return HC_OK;
    const long long m = rows * (cols - 1) + (rows - 1) * cols;
    if (m == 0) return HC_OK;
    gen_grid_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, as_stream(stream)>>>(rows, cols, m,
                                                                        (longlong2 *)d_edges);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_gen_er(int64_t n, int64_t m, uint64_t seed, int64_t *d_edges, void *stream) {
    HC_REQUIRE(n > 0 && m >= 0, HC_ERR_INVALID, "gen_er: bad sizes");
    if (m == 0) return HC_OK;
    gen_er_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, as_stream(stream)>>>((unsigned long long)n, m, seed,
                                                                       (longlong2 *)d_edges);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_gen_rmat(int scale, int64_t m, uint64_t seed, int64_t *d_edges, void *stream) {
    HC_REQUIRE(scale >= 0 && scale <= 31 && m >= 0, HC_ERR_INVALID, "gen_rmat: bad sizes");
    if (m == 0) return HC_OK;
    gen_rmat_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, as_stream(stream)>>>(scale, m, seed,
                                                                         (longlong2 *)d_edges);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

size_t hc_build_csr_workspace_bytes(int64_t n, int64_t m) {
    if (n < 0) n = 0;
    if (m < 0) m = 0;
    return csr_layout(n, n, 2 * m).total;
}

size_t hc_build_csr_rows_workspace_bytes(int64_t n, int64_t lo, int64_t hi, int64_t dir_capacity) {
    if (n < 0) n = 0;
    const long long rows = hi > lo ? hi - lo : 0;
    return csr_layout(n, rows, dir_capacity < 0 ? 0 : dir_capacity).total;
}

int hc_build_csr_rows(const int64_t *d_edges, int64_t m, int64_t n, int64_t lo, int64_t hi,
                      int64_t dir_capacity, int64_t *d_row_offsets, int32_t *d_col_indices,
                      int64_t *h_num_edges, void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(n >= 0 && n < 0x7fffffffLL && m >= 0 && h_num_edges && d_row_offsets && lo >= 0 && lo <= hi &&
                   hi <= n && dir_capacity >= 0, HC_ERR_INVALID, "build_csr: bad arguments");
    cudaStream_t st = as_stream(stream);
    const long long rows = hi - lo;
    *h_num_edges = 0;
    if (rows == 0 || m == 0) {  // graph.py:188-189
        HC_CUDA_TRY(cudaMemsetAsync(d_row_offsets, 0, 8 * (size_t)(rows + 1), st));
        HC_CUDA_TRY(cudaStreamSynchronize(st));
        return HC_OK;
    }
    const CsrLayout L = csr_layout(n, rows, dir_capacity);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "build_csr: workspace %zu < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    unsigned *deg = reinterpret_cast<unsigned *>(ws + L.deg);
    unsigned long long *off = reinterpret_cast<unsigned long long *>(ws + L.off);
    unsigned long long *cur = reinterpret_cast<unsigned long long *>(ws + L.cur);
    int *tmp = reinterpret_cast<int *>(ws + L.tmp);
    unsigned *uniq = reinterpret_cast<unsigned *>(ws + L.uniq);
    unsigned long long *ro = reinterpret_cast<unsigned long long *>(d_row_offsets);
    int *rowlist = reinterpret_cast<int *>(ws + L.rows);
    unsigned *status = reinterpret_cast<unsigned *>(ws + L.status);
    unsigned *bitmaps = reinterpret_cast<unsigned *>(ws + L.bitmaps);
    unsigned *summaries = reinterpret_cast<unsigned *>(ws + L.summaries);
    const longlong2 *edges = reinterpret_cast<const longlong2 *>(d_edges);

    HC_CUDA_TRY(cudaMemsetAsync(deg, 0, 4 * (size_t)(rows + 1), st));
    HC_CUDA_TRY(cudaMemsetAsync(status, 0, 256, st));
    HC_CUDA_TRY(cudaMemsetAsync(bitmaps, 0, 4 * (size_t)((n + 31) / 32) * (size_t)L.big_ctas, st));
    HC_CUDA_TRY(cudaMemsetAsync(summaries, 0, 4 * (size_t)((n + 1023) / 1024) * (size_t)L.big_ctas, st));
    degree_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, st>>>(edges, m, n, lo, hi, deg, status);
    HC_CHECK_LAUNCH();
    int rc = exclusive_scan(deg, rows, off, ws + L.scan, st);
    if (rc) return rc;
    unsigned long long dir = 0;
    unsigned h_status = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&dir, off + rows, sizeof dir, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaMemcpyAsync(&h_status, status, sizeof h_status, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    HC_REQUIRE(!h_status, HC_ERR_INVALID, "edge endpoint outside declared node range");  // graph.py:39-42
    HC_REQUIRE((long long)dir <= dir_capacity, HC_ERR_WORKSPACE,
               "build_csr: rows [%lld, %lld) hold %llu directed entries > capacity %lld", (long long)lo,
               (long long)hi, dir, (long long)dir_capacity);
    HC_CUDA_TRY(cudaMemcpyAsync(cur, off, 8 * (size_t)rows, cudaMemcpyDeviceToDevice, st));
    scatter_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, st>>>(edges, m, n, lo, hi, cur, tmp);
    HC_CHECK_LAUNCH();
    sort_small_rows_kernel<<<grid_cap(rows, BLOCK / 32), BLOCK, 0, st>>>(off, rows, tmp, uniq);
    HC_CHECK_LAUNCH();
    unsigned long long *totals = nullptr;
    rc = ordered_partition<2>(rows, RowBin{off}, EmitRow{}, rowlist, ws + L.part, &totals, st);
    if (rc) return rc;
    unsigned long long h_tot[2];
    HC_CUDA_TRY(cudaMemcpyAsync(h_tot, totals, sizeof h_tot, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    if (h_tot[0]) {
        sort_mid_rows_kernel<<<grid_cap((long long)h_tot[0], 1), MID_THREADS, 0, st>>>(
            off, rowlist, (long long)h_tot[0], tmp, uniq);
        HC_CHECK_LAUNCH();
    }
    if (h_tot[1]) {
        const int ctas = (int)std::min<long long>((long long)h_tot[1], L.big_ctas);
        sort_big_rows_kernel<<<ctas, BLOCK, 0, st>>>(off, rowlist + h_tot[0], (long long)h_tot[1], n, tmp,
                                                     uniq, bitmaps, summaries);
        HC_CHECK_LAUNCH();
    }
    rc = exclusive_scan(uniq, rows, ro, ws + L.scan, st);
    if (rc) return rc;
    compact_kernel<<<grid_cap(rows, BLOCK / 32), BLOCK, 0, st>>>(off, ro, tmp, rows, d_col_indices);
    HC_CHECK_LAUNCH();
    long long total = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&total, ro + rows, sizeof total, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    *h_num_edges = total;
    return HC_OK;
}

int hc_build_csr(const int64_t *d_edges, int64_t m, int64_t n, int64_t *d_row_offsets,
                 int32_t *d_col_indices, int64_t *h_num_edges, void *d_ws, size_t ws_bytes,
                 void *stream) {
    HC_REQUIRE(n >= 0 && n < 0x7fffffffLL && m >= 0, HC_ERR_INVALID, "build_csr: bad arguments");
    return hc_build_csr_rows(d_edges, m, n, 0, n, 2 * m, d_row_offsets, d_col_indices, h_num_edges, d_ws,
                             ws_bytes, stream);
}

int hc_edge_degrees(const int64_t *d_edges, int64_t m, int64_t n, int64_t *d_deg, void *stream) {
    HC_REQUIRE(n >= 0 && m >= 0 && d_deg, HC_ERR_INVALID, "edge_degrees: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_deg, 0, 8 * (size_t)std::max<int64_t>(n, 1), st));
    if (m > 0 && n > 0) {
        raw_degree_kernel<<<grid_cap(m, BLOCK), BLOCK, 0, st>>>((const longlong2 *)d_edges, m, n,
                                                                (unsigned long long *)d_deg);
        HC_CHECK_LAUNCH();
    }
    return HC_OK;
}

int hc_verify_rows(const int64_t *d_ro, const int32_t *d_ci, int64_t lo, int64_t hi, const int64_t *d_colors,
                   int64_t *d_acc, int64_t *h_bad, void *stream) {
    HC_REQUIRE(lo >= 0 && hi >= lo && d_acc && h_bad, HC_ERR_INVALID, "verify_rows: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (hi > lo) {
        verify_rows_kernel<<<grid_cap(hi - lo, BLOCK / 32), BLOCK, 0, st>>>(
            (const long long *)d_ro, d_ci, lo, hi - lo, (const long long *)d_colors, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    HC_CUDA_TRY(cudaMemcpyAsync(h_bad, d_acc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    return HC_OK;
}

int hc_verify(const int64_t *d_ro, const int32_t *d_ci, int64_t n, const int64_t *d_colors,
              int64_t *d_acc, int64_t *h_bad, void *stream) {
    HC_REQUIRE(n >= 0 && d_acc && h_bad, HC_ERR_INVALID, "verify: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (n > 0) {
        verify_kernel<<<grid_cap(n, BLOCK / 32), BLOCK, 0, st>>>(
            (const long long *)d_ro, d_ci, n, (const long long *)d_colors, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    HC_CUDA_TRY(cudaMemcpyAsync(h_bad, d_acc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    return HC_OK;
}

int hc_colors_used(const int64_t *d_colors, int64_t n, int64_t *d_acc, int64_t *h_used, void *stream) {
    HC_REQUIRE(n >= 0 && d_acc && h_used, HC_ERR_INVALID, "colors_used: bad arguments");
    *h_used = 0;
    if (n == 0) return HC_OK;  // driver.py:181-182
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, 2 * sizeof(int64_t), st));
    colors_used_kernel<<<grid_cap(n, BLOCK), BLOCK, 0, st>>>((const long long *)d_colors, n,
                                                             (unsigned long long *)d_acc);
    HC_CHECK_LAUNCH();
    long long h[2];
    HC_CUDA_TRY(cudaMemcpyAsync(h, d_acc, sizeof h, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    HC_REQUIRE(h[1] == 0, HC_ERR_UNCOLORED, "invalid coloring: uncolored node (color 0) present");
    *h_used = h[0];
    return HC_OK;
}

int hc_narrow_i64_i32(const int64_t *d_in, int32_t *d_out, int64_t count, void *stream) {
    HC_REQUIRE(count >= 0, HC_ERR_INVALID, "narrow: negative count");
    if (count == 0) return HC_OK;
    narrow_kernel<<<grid_cap(count, BLOCK), BLOCK, 0, as_stream(stream)>>>((const long long *)d_in,
                                                                           d_out, count);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

int hc_csr_check_lower_first(const int64_t *d_ro, const int32_t *d_ci, int64_t n, int64_t *d_acc,
                             int64_t *h_bad_rows, void *stream) {
    HC_REQUIRE(n >= 0 && d_acc && h_bad_rows, HC_ERR_INVALID, "check_lower_first: bad arguments");
    cudaStream_t st = as_stream(stream);
    HC_CUDA_TRY(cudaMemsetAsync(d_acc, 0, sizeof(int64_t), st));
    if (n > 0) {
        lower_first_check_kernel<<<grid_cap(n, BLOCK / 32), BLOCK, 0, st>>>(
            (const long long *)d_ro, d_ci, n, (unsigned long long *)d_acc);
        HC_CHECK_LAUNCH();
    }
    HC_CUDA_TRY(cudaMemcpyAsync(h_bad_rows, d_acc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    return HC_OK;
}

int hc_csr_partition_lower_first(const int64_t *d_ro, const int32_t *d_ci_in, int32_t *d_ci_out, int64_t n,
                                 void *stream) {
    HC_REQUIRE(n >= 0 && d_ci_in != d_ci_out, HC_ERR_INVALID, "partition_lower_first: bad arguments");
    if (n == 0) return HC_OK;
    lower_first_partition_kernel<<<grid_cap(n, BLOCK / 32), BLOCK, 0, as_stream(stream)>>>(
        (const long long *)d_ro, d_ci_in, d_ci_out, n);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

}  // extern "C"
