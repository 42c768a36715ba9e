// hcb_partition.cuh -- order-preserving multi-bin partition (stream compaction)
// of an index range, in three passes: per-tile bin counts, one-CTA exclusive
// scan of the (bin-major) tile counts, ordered scatter.  Used for the solver's
// static degree bins, the worklist swap_and_sort and the CSR build.
//
// Tile = PART_THREADS * PART_ITEMS consecutive indices; each thread owns
// PART_ITEMS consecutive indices (blocked arrangement) so thread order equals
// index order and the output of every bin is ascending in the input index.
#pragma once

#include "hcb_common.cuh"

namespace hcb {

constexpr int PART_THREADS = 256;
constexpr int PART_ITEMS = 8;
constexpr long long PART_TILE = PART_THREADS * PART_ITEMS;
constexpr int PART_SCAN_THREADS = 1024;

inline long long part_tiles(long long count) { return (count + PART_TILE - 1) / PART_TILE; }

// scratch: NB * tiles uint32 counts + NB uint64 totals
inline size_t part_scratch_bytes(int nb, long long count) {
    return align_up(sizeof(unsigned long long) * (size_t)nb * (size_t)part_tiles(count), 256) +
           align_up(sizeof(unsigned long long) * (size_t)nb, 256);
}

template <int NB, class Classify>
__global__ void __launch_bounds__(PART_THREADS) part_count_kernel(long long count, Classify cls,
                                                                  unsigned long long *tile_counts,
                                                                  long long tiles) {
    __shared__ unsigned s_cnt[NB];
    if (threadIdx.x < NB) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * PART_TILE + (long long)threadIdx.x * PART_ITEMS;
    unsigned c[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) c[b] = 0;
#pragma unroll
    for (int j = 0; j < PART_ITEMS; ++j) {
        long long i = base + j;
        if (i < count) {
            int b = cls(i);
#pragma unroll
            for (int q = 0; q < NB; ++q) c[q] += (b == q);
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        unsigned w = warp_sum(c[b]);
        if (lane_id() == 0 && w) atomicAdd(&s_cnt[b], w);
    }
    __syncthreads();
    if (threadIdx.x < NB) tile_counts[(long long)threadIdx.x * tiles + blockIdx.x] = s_cnt[threadIdx.x];
}

// exclusive scan over NB*tiles values in place; totals[b] = elements of bin b
__global__ void __launch_bounds__(PART_SCAN_THREADS) part_scan_kernel(unsigned long long *vals,
                                                                      long long len, int nb,
                                                                      long long tiles,
                                                                      unsigned long long *totals);

template <int NB, class Classify, class Emit, class OutT>
__global__ void __launch_bounds__(PART_THREADS) part_write_kernel(long long count, Classify cls,
                                                                  Emit emit,
                                                                  const unsigned long long *tile_offsets,
                                                                  long long tiles, OutT *out) {
    static_assert(NB <= 3, "packed 21-bit scan supports up to 3 bins");
    __shared__ unsigned long long s_warp[PART_THREADS / 32];
    const long long base = (long long)blockIdx.x * PART_TILE + (long long)threadIdx.x * PART_ITEMS;
    int bins[PART_ITEMS];
    unsigned long long packed = 0;
#pragma unroll
    for (int j = 0; j < PART_ITEMS; ++j) {
        long long i = base + j;
        int b = i < count ? cls(i) : -1;
        bins[j] = b;
        if (b >= 0) packed += 1ull << (21 * b);
    }
    // block exclusive scan of the packed per-bin counts
    unsigned long long incl = warp_incl_scan(packed);
    const unsigned warp = threadIdx.x >> 5;
    if (lane_id() == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long v = lane_id() < PART_THREADS / 32 ? s_warp[lane_id()] : 0;
        unsigned long long vi = warp_incl_scan(v);
        if (lane_id() < PART_THREADS / 32) s_warp[lane_id()] = vi - v;
    }
    __syncthreads();
    unsigned long long excl = incl - packed + s_warp[warp];
    unsigned long long pos[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b)
        pos[b] = tile_offsets[(long long)b * tiles + blockIdx.x] + ((excl >> (21 * b)) & 0x1fffffull);
#pragma unroll
    for (int j = 0; j < PART_ITEMS; ++j) {
        int b = bins[j];
#pragma unroll
        for (int q = 0; q < NB; ++q)
            if (b == q) out[pos[q]++] = emit(base + j);
    }
}

// Host driver.  scratch must hold part_scratch_bytes(NB, count).  After the
// call, `totals` (device, NB uint64) holds the per-bin sizes and bin b starts
// at sum(totals[0..b)) in `out`.
template <int NB, class Classify, class Emit, class OutT>
int ordered_partition(long long count, Classify cls, Emit emit, OutT *out, void *scratch,
                      unsigned long long **totals_out, cudaStream_t st) {
    const long long tiles = part_tiles(count);
    unsigned long long *tile_counts = reinterpret_cast<unsigned long long *>(scratch);
    unsigned long long *totals = reinterpret_cast<unsigned long long *>(
        reinterpret_cast<char *>(scratch) +
        align_up(sizeof(unsigned long long) * (size_t)NB * (size_t)tiles, 256));
    if (totals_out) *totals_out = totals;
    if (count == 0) {
        HC_CUDA_TRY(cudaMemsetAsync(totals, 0, sizeof(unsigned long long) * NB, st));
        return HC_OK;
    }
    part_count_kernel<NB><<<(unsigned)tiles, PART_THREADS, 0, st>>>(count, cls, tile_counts, tiles);
    HC_CHECK_LAUNCH();
    part_scan_kernel<<<1, PART_SCAN_THREADS, 0, st>>>(tile_counts, (long long)NB * tiles, NB, tiles,
                                                     totals);
    HC_CHECK_LAUNCH();
    part_write_kernel<NB><<<(unsigned)tiles, PART_THREADS, 0, st>>>(count, cls, emit, tile_counts,
                                                                    tiles, out);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

}  // namespace hcb

namespace hcb {

// ---------------------------------------------------------------------------
// Bucket sort of an index range by a small key (K <= 32 buckets): per-tile
// histograms, one-CTA scan (bucket-major), scatter through shared-memory
// cursors.  Buckets come out in key order; within a bucket, tiles keep their
// order (positions inside one tile follow shared-memory atomics).
// ---------------------------------------------------------------------------
template <int K, class Key>
__global__ void __launch_bounds__(PART_THREADS) bucket_count_kernel(long long count, Key key,
                                                                    unsigned long long *tile_counts,
                                                                    long long tiles) {
    __shared__ unsigned s_cnt[K];
    for (int i = threadIdx.x; i < K; i += PART_THREADS) s_cnt[i] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * PART_TILE;
    for (int j = 0; j < PART_ITEMS; ++j) {
        const long long i = base + (long long)j * PART_THREADS + threadIdx.x;
        if (i < count) {
            const int b = key(i);
            if (b >= 0) atomicAdd(&s_cnt[b], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < K; b += PART_THREADS)
        tile_counts[(long long)b * tiles + blockIdx.x] = s_cnt[b];
}

template <int K, class Key, class Emit, class OutT>
__global__ void __launch_bounds__(PART_THREADS) bucket_scatter_kernel(long long count, Key key, Emit emit,
                                                                      const unsigned long long *tile_offsets,
                                                                      long long tiles, OutT *out) {
    __shared__ unsigned long long s_cur[K];
    for (int b = threadIdx.x; b < K; b += PART_THREADS)
        s_cur[b] = tile_offsets[(long long)b * tiles + blockIdx.x];
    __syncthreads();
    const long long base = (long long)blockIdx.x * PART_TILE;
    for (int j = 0; j < PART_ITEMS; ++j) {
        const long long i = base + (long long)j * PART_THREADS + threadIdx.x;
        const int b = i < count ? key(i) : -1;
        // warp-aggregated cursor bump: one shared atomic per (warp, bucket)
        // instead of one per node (a tile of one bucket serialised 256
        // same-address atomics per step)
        const unsigned peers = __match_any_sync(FULL, b);
        if (b >= 0) {
            const int leader = __ffs(peers) - 1;
            unsigned long long at = 0;
            if ((int)lane_id() == leader) at = atomicAdd(&s_cur[b], (unsigned long long)__popc(peers));
            at = __shfl_sync(peers, at, leader);
            out[at + __popc(peers & lanemask_lt())] = emit(i);
        }
    }
}

template <int K, class Key, class Emit, class OutT>
int bucket_sort(long long count, Key key, Emit emit, OutT *out, void *scratch,
                unsigned long long **totals_out, cudaStream_t st) {
    const long long tiles = part_tiles(count);
    unsigned long long *tile_counts = reinterpret_cast<unsigned long long *>(scratch);
    unsigned long long *totals = reinterpret_cast<unsigned long long *>(
        reinterpret_cast<char *>(scratch) +
        align_up(sizeof(unsigned long long) * (size_t)K * (size_t)tiles, 256));
    if (totals_out) *totals_out = totals;
    if (count == 0) {
        HC_CUDA_TRY(cudaMemsetAsync(totals, 0, sizeof(unsigned long long) * K, st));
        return HC_OK;
    }
    bucket_count_kernel<K><<<(unsigned)tiles, PART_THREADS, 0, st>>>(count, key, tile_counts, tiles);
    HC_CHECK_LAUNCH();
    part_scan_kernel<<<1, PART_SCAN_THREADS, 0, st>>>(tile_counts, (long long)K * tiles, K, tiles, totals);
    HC_CHECK_LAUNCH();
    bucket_scatter_kernel<K><<<(unsigned)tiles, PART_THREADS, 0, st>>>(count, key, emit, tile_counts,
                                                                      tiles, out);
    HC_CHECK_LAUNCH();
    return HC_OK;
}

}  // namespace hcb
