// hcb_solve.cu -- host side of the device-resident IPGC solve (hc_solve):
// per-solve preprocessing, the format / kernel choice, the cooperative launch
// and the C-ABI (include/hcb.h).  The device code is hcb_solve_dev.cuh; the
// solve_kernel instantiations live in hcb_solve_inst.cu (one object per group).
#include "hcb_solve_dev.cuh"

namespace hcb {
namespace solve {

#define HC_EXTERN_INST(OffT, F, ST) extern template const void *kernel_ptr<OffT, F, ST>();
HC_INST_ALL(HC_EXTERN_INST)
#undef HC_EXTERN_INST

// Static lists: nodes bucket-sorted by a degree key.  Keys 0-2 are bins 0-2;
// bin 3 and the hubs are split into power-of-two degree buckets in
// DESCENDING order, so chunks of those bins hold nodes of similar degree
// (balanced warps) and the heaviest nodes are handed out first.
constexpr int NKEY = 15;
__host__ __device__ constexpr int key_bin(int key) {
    return key <= 2 ? key : key <= 8 ? 3 : 4;
}
struct DegreeKey {
    const long long *ro;
    __device__ int operator()(long long i) const {
        const long long d = ro[i + 1] - ro[i];
        const int b = bin_of_degree(d);
        if (b <= 2) return b;
        const int lg = 64 - __clzll(d - 1);  // ceil(log2 d): 65..128 -> 7, 2049..4096 -> 12
        if (b == 3) return 3 + (12 - lg);    // keys 3..8
        return 9 + max(0, 18 - lg);          // hubs: >= 2^17+1 -> 9 ... 4097..8192 -> 14
    }
};
struct EmitI32 {
    long long lo;  // first owned node (multi-GPU), 0 on one GPU
    __device__ int operator()(long long i) const { return (int)(lo + i); }
};

__global__ void copy_totals_kernel(const unsigned long long *tot, Ctrl *c) {
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBIN; ++b) c->nstat[b] = 0;
        for (int k = 0; k < NKEY; ++k) c->nstat[key_bin(k)] += tot[k];
    }
}

__global__ void narrow_offsets_kernel(const long long *ro, int *ro32, long long count) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        ro32[i] = (int)ro[i];
}

// int16 delta columns ci16[k] = ci[k] - u; sets *bad when some |v-u| >= 2^15
// (then the absolute int32 columns are used).  Thread per row for rows of
// up to 32 entries, the whole warp for longer ones (one thread walking a
// 9725-entry hub row cost RMAT-16 1.1 ms per solve); every warp stops at the
// first violation anywhere.  With ell != nullptr the same pass writes the ELL4 word
// of every row of degree <= 4 (4 int16 deltas, row order, 0-padded) and sets
// *ell_bad at the first row of degree > 4 (then the ELL4 kernel is not used).
// Rows of more than 32 entries are only listed here (big_rows, *nbig) and
// converted by delta_columns_big_kernel, one CTA per row: the hubs of an RMAT
// graph have the lowest ids, so one warp walking its own 32 rows held the
// whole pass (RMAT-16: nodes 0..31 hold 58.8 K entries, 139 us).
__global__ void delta_columns_kernel(const long long *ro, const int *ci, long long lo, long long hi,
                                     short *ci16, unsigned *bad, unsigned long long *ell, unsigned *ell_bad,
                                     int *big_rows, unsigned *nbig) {
    const unsigned lane = lane_id();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = lo + (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < hi; base += stride) {
        if (__any_sync(FULL, *(volatile unsigned *)bad != 0u)) return;  // warp-uniform
        const long long u = base + lane;
        const bool valid = u < hi;
        const long long b = valid ? ro[u] : 0, e = valid ? ro[u + 1] : 0;
        const bool big = e - b > 32;
        bool fail = false;
        if (valid && !big) {
            const bool fits = e - b <= 4;
            unsigned long long w = 0;
            for (long long k = b; k < e; ++k) {
                const long long d = (long long)ci[k] - u;
                if (d < -32768 || d > 32767) {
                    fail = true;
                    break;
                }
                ci16[k] = (short)d;
                if (fits) w |= (unsigned long long)(unsigned short)(short)d << (16 * (k - b));
            }
            if (ell && !fail) {
                if (fits) ell[u - lo] = w;
                else if (!*(volatile unsigned *)ell_bad) atomicOr(ell_bad, 1u);
            }
        }
        // rows longer than 32 entries: listed for delta_columns_big_kernel
        const unsigned bigs = __ballot_sync(FULL, valid && big);
        if (bigs) {
            if (ell && !*(volatile unsigned *)ell_bad && lane == 0) atomicOr(ell_bad, 1u);
            unsigned at = 0;
            if (lane == 0) at = atomicAdd(nbig, (unsigned)__popc(bigs));
            at = __shfl_sync(FULL, at, 0);
            if (valid && big) big_rows[at + __popc(bigs & lanemask_lt())] = (int)u;
        }
        if (__any_sync(FULL, fail)) {
            if (lane == 0) atomicOr(bad, 1u);
            return;
        }
    }
}

// the listed rows of more than 32 entries, one CTA per row (no barriers: a
// CTA may stop part-way once some row failed)
__global__ void delta_columns_big_kernel(const long long *ro, const int *ci, const int *big_rows,
                                         const unsigned *nbig, short *ci16, unsigned *bad) {
    const unsigned nr = *nbig;
    for (unsigned r = blockIdx.x; r < nr; r += gridDim.x) {
        if (*(volatile unsigned *)bad) return;
        const long long u = big_rows[r];
        const long long b = ro[u], e = ro[u + 1];
        bool fail = false;
        for (long long k = b + threadIdx.x; k < e; k += blockDim.x) {
            const long long d = (long long)ci[k] - u;
            if (d < -32768 || d > 32767) fail = true;
            else ci16[k] = (short)d;
        }
        if (fail) atomicOr(bad, 1u);
    }
}

// (row offset << 16 | degree) of every static list entry (degrees above
// 0xffff -- hubs only, which never read it -- are clamped)
__global__ void fill_od_kernel(const long long *ro, const int *stat, long long count, unsigned long long *od) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const int u = stat[i];
        const long long b = ro[u], d = ro[u + 1] - b;
        od[i] = ((unsigned long long)b << 16) | (unsigned long long)(d < 0xffff ? d : 0xffff);
    }
}

// max degree over all nodes (the multi-GPU state-word format must agree on
// every rank, so it is decided from the whole graph)
__global__ void max_degree_kernel(const long long *ro, long long n, unsigned long long *out) {
    unsigned long long d = 0;
    for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x)
        d = max(d, (unsigned long long)(ro[u + 1] - ro[u]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = max(d, __shfl_xor_sync(FULL, d, o));
    if (lane_id() == 0 && d) atomicMax(out, d);
}

// multi-GPU: per owned node the mask of the ranks holding a neighbour, and the
// boundary zones (longest prefix / suffix of the owned range that contains a
// node read by a lower / higher rank).  Warp per node.
__global__ void mg_boundary_kernel(const long long *ro, const int *ci, const long long *bounds, int world,
                                   int rank, unsigned char *mask, unsigned long long *zones) {
    __shared__ long long sb[MG_MAX_WORLD + 1];
    if (threadIdx.x <= (unsigned)world) sb[threadIdx.x] = bounds[threadIdx.x];
    __syncthreads();
    const long long lo = sb[rank], hi = sb[rank + 1];
    const unsigned lane = lane_id();
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long u = lo + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5); u < hi; u += nwarps) {
        unsigned m = 0;
        for (long long k = ro[u] + lane; k < ro[u + 1]; k += 32) {
            const long long v = ci[k];
            if (v >= lo && v < hi) continue;
            int q = 0;
            while (q + 1 < world && v >= sb[q + 1]) ++q;
            m |= 1u << q;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m |= __shfl_xor_sync(FULL, m, o);
        if (lane == 0) {
            mask[u - lo] = (unsigned char)m;
            if (m) atomicAdd(&zones[2], (unsigned long long)__popc(m));
            if (m & ((1u << rank) - 1u)) atomicMax(&zones[0], (unsigned long long)(u - lo + 1));
            if (m >> (rank + 1)) atomicMax(&zones[1], (unsigned long long)(hi - u));
        }
    }
}

// worst-case segmented capacity of a bin with `cnt` static nodes
inline size_t seg_capacity(long long cnt) {
    return (size_t)cnt + (size_t)cnt / MAXSEG + 2 * BLOCK * NPT;
}

struct Layout {
    size_t ctrl, x, stat, dyn[2][NBIN], stat_od, dyn_od[2][NSEG_BINS], ro32, ci16, hub_acc, part, bnd, ptrs,
        maxdeg, fb0, fbx, fbx_bytes, ell, lc, lcnt, total;
};

// The dynamic bin regions depend on the bin sizes, which are only known on
// the device; size each for the whole owned node count (upper bound of every
// bin).  The control block comes first (hc_mg_wait finds it there).  The
// multi-GPU layout has no state words (they live in the peer-mapped shared
// region) but boundary flags and the peer pointer tables.
static Layout layout(long long n, long long m, long long nown, bool mg) {
    Layout L;
    size_t o = 0;
    L.ctrl = o; o = align_up(o + sizeof(Ctrl), 256);
    L.x = o; o = align_up(o + (mg ? 0 : 4 * (size_t)n), 256);
    L.stat = o; o = align_up(o + 4 * (size_t)nown, 256);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NBIN; ++b) {
            L.dyn[p][b] = o;
            o = align_up(o + 4 * (b == BIN_HUB ? (size_t)nown : seg_capacity(nown)), 256);
        }
    L.stat_od = o; o = align_up(o + 8 * (size_t)nown, 256);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NSEG_BINS; ++b) {
            L.dyn_od[p][b] = o;
            o = align_up(o + 8 * seg_capacity(nown), 256);
        }
    L.ro32 = o; o = align_up(o + 4 * (size_t)(nown + 1), 256);
    L.ci16 = o; o = align_up(o + (m < 0x7fffffffLL ? 2 * (size_t)m : 0) + 256, 256);
    L.hub_acc = o; o = align_up(o + sizeof(HubAcc) * MAX_SPLIT_SLOTS, 256);
    L.part = o; o = align_up(o + part_scratch_bytes(NKEY, nown), 256);
    L.bnd = o; o = align_up(o + (mg ? (size_t)nown : 0), 256);
    L.ptrs = o; o = align_up(o + (mg ? 2 * sizeof(void *) * MG_MAX_WORLD + 8 * (MG_MAX_WORLD + 1) + 24 : 0), 256);
    L.maxdeg = o; o = align_up(o + 8, 256);
    // forbidden-color bitmaps (single GPU): fb0 one word per node, fbx
    // floor(deg/32) words per node at ro >> 5 (+ slack for the group reads)
    L.fb0 = o; o = align_up(o + (mg ? 0 : 4 * (size_t)n), 256);
    L.fbx_bytes = mg ? 0 : 4 * ((size_t)(m >> 5) + 64);
    L.fbx = o; o = align_up(o + L.fbx_bytes, 256);
    // ELL4 rows (single GPU, every degree <= 4): 8 bytes per node
    L.ell = o; o = align_up(o + (mg ? 0 : 8 * (size_t)n), 256);
    // live lower lists (single GPU): one int32 per half-edge + a count per node
    L.lc = o; o = align_up(o + (mg ? 0 : 4 * (size_t)m), 256);
    L.lcnt = o; o = align_up(o + (mg ? 0 : 4 * (size_t)n), 256);
    L.total = o;
    return L;
}

template <class F32_, class F16_, class F16D_, class F32D_, bool STATS>
static const void *pick(bool narrow, bool x16, bool c16) {
    static_assert(!F16D_::ell, "ELL4 kernels are picked by pick_ell");
    if (!narrow) return x16 ? kernel_ptr<long long, F16_, STATS>() : kernel_ptr<long long, F32_, STATS>();
    if (x16 && c16) return kernel_ptr<int, F16D_, STATS>();
    if (x16) return kernel_ptr<int, F16_, STATS>();
    if (c16) return kernel_ptr<int, F32D_, STATS>();
    return kernel_ptr<int, F32_, STATS>();
}

// the instantiation for (offset width, state width, column format, bin-0
// only, stats, ELL4 rows).  int64 offsets (m >= 2^31) keep 32-bit words.
static const void *select_kernel(bool narrow, bool x16, bool c16, bool stats, bool small = false,
                                 bool plain = false, bool ell = false, bool live = false, bool x8 = false) {
    if (!narrow) x16 = c16 = x8 = false;
    if (x8 && !stats && !live && !small) {  // 8-bit state words (general kernel, int32 offsets, no statistics)
        return plain ? (c16 ? kernel_ptr<int, PF8D, false>() : kernel_ptr<int, PF8, false>())
                     : (c16 ? kernel_ptr<int, F8D, false>() : kernel_ptr<int, F8, false>());
    }
    if (live && !small && !plain)
        return stats ? pick<LF32, LF16, LF16D, LF32D, true>(narrow, x16, c16)
                     : pick<LF32, LF16, LF16D, LF32D, false>(narrow, x16, c16);
    if (small && c16 && ell) {  // ELL4 rows imply int32 offsets and delta columns
        if (plain) return x16 ? kernel_ptr<int, PSEF16D, false>() : kernel_ptr<int, PSEF32D, false>();
        if (stats) return x16 ? kernel_ptr<int, SEF16D, true>() : kernel_ptr<int, SEF32D, true>();
        return x16 ? kernel_ptr<int, SEF16D, false>() : kernel_ptr<int, SEF32D, false>();
    }
    if (plain)  // bench-only Plain baseline (no statistics build)
        return small ? pick<PSF32, PSF16, PSF16D, PSF32D, false>(narrow, x16, c16)
                     : pick<PF32, PF16, PF16D, PF32D, false>(narrow, x16, c16);
    if (small)
        return stats ? pick<SF32, SF16, SF16D, SF32D, true>(narrow, x16, c16)
                     : pick<SF32, SF16, SF16D, SF32D, false>(narrow, x16, c16);
    return stats ? pick<F32, F16, F16D, F32D, true>(narrow, x16, c16)
                 : pick<F32, F16, F16D, F32D, false>(narrow, x16, c16);
}

// multi-GPU instantiations (no per-round edge statistics)
static const void *select_kernel_mg(bool narrow, bool x16, bool c16, bool small = false) {
    if (small) return pick<SMF32, SMF16, SMF16D, SMF32D, false>(narrow, x16, c16);
    return pick<MF32, MF16, MF16D, MF32D, false>(narrow, x16, c16);
}

static int occupancy_of(const void *fn) {
    // cached per (kernel, device, calling thread): the query costs host time
    // on every solve, while the GPU waits for the launch (small graphs)
    static thread_local std::unordered_map<const void *, int> cache[8];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
    if (dev >= 0 && dev < 8) {
        const auto it = cache[dev].find(fn);
        if (it != cache[dev].end()) return it->second;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BLOCK, 0) != cudaSuccess) return 0;
    if (dev >= 0 && dev < 8) cache[dev][fn] = per_sm;
    return per_sm;
}

static int occupancy() {
    int lo = 1 << 30;
    for (bool n : {false, true})
        for (bool x : {false, true})
            for (bool c : {false, true}) lo = std::min(lo, occupancy_of(select_kernel(n, x, c, false)));
    return lo;
}

// format overrides (tests / experiments): force int64 offsets, forbid the
// 16-bit state word, forbid 16-bit delta columns, the multi-GPU exchange mode.
// Per host thread: a knob set by one caller never changes another thread's solves.
static thread_local int g_no_x8 = 0;
static thread_local int g_force_wide = 0, g_no_x16 = 0, g_no_c16 = 0, g_no_small = 0, g_mg_exchange = 0,
                        g_no_ell = 0, g_live = -1;

// Per-solve preprocessing shared by hc_solve and hc_mg_solve, for the owned
// range [lo, lo + nown): fresh control block, static degree-bucketed lists,
// int32 offsets, int16 delta columns; reads back the bucket totals, the
// delta-column verdict and (on request) the owned rows' max degree.
// d_row_offsets holds the owned rows only (row r = node lo+r: the whole graph
// on one GPU, the rank's shard on several); the kernels index it by global
// node id through the shifted pointer ro_v = d_row_offsets - lo.
struct Prep {
    unsigned long long tot[NKEY];
    unsigned long long *d_totals;
    bool narrow, c16_ok, ell_ok;
    unsigned long long max_degree;
};

// ell: the ELL4 row array to fill (single GPU), nullptr on a multi-GPU rank
// workspace pointers of a solve (prepare; hc_solve_launch re-binds a planned workspace)
static void bind_params(Params &P, const Layout &L, char *ws, const int64_t *d_row_offsets, bool narrow) {
    P.ctrl = reinterpret_cast<Ctrl *>(ws + L.ctrl);
    P.hub_acc = reinterpret_cast<HubAcc *>(ws + L.hub_acc);
    P.stat = reinterpret_cast<int *>(ws + L.stat);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NBIN; ++b) P.dyn[p][b] = reinterpret_cast<int *>(ws + L.dyn[p][b]);
    P.stat_od = reinterpret_cast<unsigned long long *>(ws + L.stat_od);
    for (int p = 0; p < 2; ++p)
        for (int b = 0; b < NSEG_BINS; ++b) P.dyn_od[p][b] = reinterpret_cast<unsigned long long *>(ws + L.dyn_od[p][b]);
    P.fmt_overflow = &P.ctrl->fmt_overflow;
    const long long *ro_v = reinterpret_cast<const long long *>(d_row_offsets) - P.lo;  // indexed by global node id
    P.ro = narrow ? (const void *)(reinterpret_cast<const int *>(ws + L.ro32) - P.lo) : (const void *)ro_v;
    P.ci16 = reinterpret_cast<const short *>(ws + L.ci16);
}

static int prepare(Params &P, const Layout &L, char *ws, const int64_t *d_row_offsets, long long n,
                   long long m, bool want_maxdeg, Prep &out, cudaStream_t st,
                   unsigned long long *ell = nullptr) {
    (void)n;
    const bool narrow = m < 0x7fffffffLL && !g_force_wide;
    out.narrow = narrow;
    bind_params(P, L, ws, d_row_offsets, narrow);
    HC_CUDA_TRY(cudaMemsetAsync(P.ctrl, 0, offsetof(Ctrl, segcnt), st));
    HC_CUDA_TRY(cudaMemsetAsync(P.hub_acc, 0, sizeof(HubAcc) * MAX_SPLIT_SLOTS, st));
    const long long *ro_loc = reinterpret_cast<const long long *>(d_row_offsets);
    const long long *ro_v = ro_loc - P.lo;  // indexed by global node id (owned nodes only)
    // static degree-bucketed lists of the owned nodes (bins contiguous, see DegreeKey)
    int rc = bucket_sort<NKEY>(P.nown, DegreeKey{ro_loc}, EmitI32{P.lo}, P.stat, ws + L.part,
                               &out.d_totals, st);
    if (rc != HC_OK) return rc;
    const int sms = std::max(1, num_sms());
    copy_totals_kernel<<<1, 32, 0, st>>>(out.d_totals, P.ctrl);
    HC_CHECK_LAUNCH();
    if (P.nown > 0) {
        fill_od_kernel<<<sms * 8, 256, 0, st>>>(ro_v, P.stat, P.nown, P.stat_od);
        HC_CHECK_LAUNCH();
    }
    if (narrow) {
        narrow_offsets_kernel<<<sms * 4, 256, 0, st>>>(ro_loc, reinterpret_cast<int *>(ws + L.ro32), P.nown + 1);
        HC_CHECK_LAUNCH();
    }
    // int16 delta columns of the owned rows when every |v - u| < 2^15
    // (behind the int16 columns, 16-byte aligned: a rank's shard can hold an odd number of half-edges)
    unsigned *bad = reinterpret_cast<unsigned *>(ws + L.ci16 + (narrow ? align_up(2 * (size_t)m, 16) : 0));
    unsigned *ell_bad = bad + 1;
    unsigned *nbig = bad + 2;  // rows of > 32 entries, listed in the (not yet used) dynamic list of bin 0
    HC_CUDA_TRY(cudaMemsetAsync(bad, 0, 3 * sizeof(unsigned), st));
    P.ell = ell;
    if (narrow && m > 0 && P.nown > 0) {
        int *big_rows = reinterpret_cast<int *>(ws + L.dyn[1][0]);
        delta_columns_kernel<<<sms * 8, 256, 0, st>>>(ro_v, P.ci, P.lo, P.lo + P.nown,
                                                      reinterpret_cast<short *>(ws + L.ci16), bad, ell, ell_bad,
                                                      big_rows, nbig);
        HC_CHECK_LAUNCH();
        delta_columns_big_kernel<<<sms * 4, 256, 0, st>>>(ro_v, P.ci, big_rows, nbig,
                                                          reinterpret_cast<short *>(ws + L.ci16), bad);
        HC_CHECK_LAUNCH();
    }
    unsigned long long *d_maxdeg = reinterpret_cast<unsigned long long *>(ws + L.maxdeg);
    out.max_degree = 0;
    if (want_maxdeg) {
        HC_CUDA_TRY(cudaMemsetAsync(d_maxdeg, 0, 8, st));
        max_degree_kernel<<<sms * 4, 256, 0, st>>>(ro_loc, P.nown, d_maxdeg);
        HC_CHECK_LAUNCH();
    }
    unsigned h_bad[2] = {1, 1};
    HC_CUDA_TRY(cudaMemcpyAsync(out.tot, out.d_totals, sizeof out.tot, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaMemcpyAsync(h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, st));
    if (want_maxdeg)
        HC_CUDA_TRY(cudaMemcpyAsync(&out.max_degree, d_maxdeg, 8, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    out.c16_ok = (HC_FMT16 != 0) && !g_no_c16 && narrow && m > 0 && h_bad[0] == 0;
    out.ell_ok = out.c16_ok && ell != nullptr && h_bad[1] == 0 && !g_no_ell;
    return HC_OK;
}

// the multi-GPU shared region of a rank: state-word replica, then mailbox
inline size_t mg_x_bytes(long long n) { return align_up(4 * (size_t)std::max(n, 1LL), 256); }

// prepared multi-GPU launches, keyed by workspace (hc_mg_prepare -> hc_mg_launch)
struct MgLaunch {
    Params P;
    const void *fn;
    bool regular;
};
static std::mutex g_mg_mu;
static std::unordered_map<void *, MgLaunch> g_mg_prepared;

// Cooperative launch of the solve kernel with the state-word array as an L2
// persisting access-policy window: the neighbour-word gathers are the reuse
// the streamed column ids would otherwise evict (HC_L2_PERSIST=0 disables).
#ifndef HC_L2_FRAC
#define HC_L2_FRAC 3   // the window only when the array is below L2 / HC_L2_FRAC
#endif
#ifndef HC_L2_PERSIST
#define HC_L2_PERSIST 1
#endif
static thread_local int g_no_l2_window = 0;  // hc_solve_set_l2_window(0): never set a window

// Demotes the solve's persisting lines back to normal: every line of the
// window is touched under an access-policy window with hitProp = Normal.
// Stream-ordered and scoped to the state-word array -- unlike
// cudaCtxResetPersistingL2Cache it leaves the caller's own persisting lines
// alone and needs no host synchronisation.
__global__ void l2_demote_kernel(const uint4 *x, long long n16, unsigned *sink) {
    unsigned acc = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
        acc ^= __ldcg(x + i).x;
    if (acc == 0x9e3779b9u && sink) *sink = acc;  // keeps the loads
}

static cudaError_t l2_demote(void *x, size_t xbytes, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max(1, num_sms() * 4));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = x;
    attr[0].val.accessPolicyWindow.num_bytes = xbytes;
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint4 *p = reinterpret_cast<const uint4 *>(x);
    long long n16 = (long long)(xbytes / 16);
    unsigned *sink = nullptr;
    void *args[] = {&p, &n16, &sink};
    return cudaLaunchKernelExC(&cfg, (const void *)l2_demote_kernel, args);
}

// *windowed: the launch carried the persisting window (the caller demotes it
// after the solve with l2_demote)
static cudaError_t launch_persistent(const void *fn, unsigned nblocks, void **args, cudaStream_t st, void *x,
                                     size_t xbytes, bool cooperative, bool *windowed = nullptr) {
    if (windowed) *windowed = false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblocks);
    cfg.blockDim = dim3(BLOCK);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (cooperative) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    // per-device state (a process may drive several GPUs)
    constexpr int MAXDEV = 64;
    static size_t persist_max_of[MAXDEV], limit_set_of[MAXDEV], l2_of[MAXDEV];
    static bool queried[MAXDEV];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAXDEV) dev = -1;
    if (dev >= 0 && !queried[dev]) {
        int v = 0;
        persist_max_of[dev] =
            cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev) == cudaSuccess ? (size_t)v : 0;
        v = 0;
        l2_of[dev] = cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess ? (size_t)v : 0;
        queried[dev] = true;
    }
    const size_t persist_max = dev >= 0 ? persist_max_of[dev] : 0;
    const size_t l2 = dev >= 0 ? l2_of[dev] : 0;
    // only when the whole array fits the set-aside AND leaves most of L2 to
    // the rest (the forbidden-color bitmaps, the streamed columns): a window
    // over a third of L2 or more measured slower (ER-2^25's 67 MB of words:
    // 73.4 ms without, 90.8 ms with; a partial window over RMAT-26's 134 MB
    // 1533 -> 1547 ms); small arrays stay in L2 anyway, there the window only
    // adds driver calls (RMAT-16: 2.9 -> 3.9 ms).  Grid4096 (33.5 MB of
    // words): 464 -> 443 ms with the window
    if (HC_L2_PERSIST && !g_no_l2_window && persist_max > 0 && xbytes >= ((size_t)16 << 20) &&
        xbytes <= persist_max && HC_L2_FRAC * xbytes < l2) {
        const size_t want = xbytes;
        cudaError_t e = cudaSuccess;
        if (limit_set_of[dev] != want) {  // exactly the array (a larger set-aside slowed the grid 590 -> 605 ms)
            e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
            if (e == cudaSuccess) limit_set_of[dev] = want;
        }
        if (e == cudaSuccess) {
            attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
            attr[na].val.accessPolicyWindow.base_ptr = x;
            attr[na].val.accessPolicyWindow.num_bytes = xbytes;
            attr[na].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)want / (double)xbytes);
            attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            ++na;
            if (windowed) *windowed = true;
        } else {
            cudaGetLastError();  // not supported here: plain launch
        }
    } else if (dev >= 0 && limit_set_of[dev] != 0 && !g_no_l2_window) {
        // a solve without a window gives the set-aside back: a grid solve's
        // 33.5 MB left in place made a later ER-2^25 solve in the same process
        // 46.7 -> 53.3 ms
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0) == cudaSuccess) limit_set_of[dev] = 0;
        else cudaGetLastError();
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

// driver API entry point (no -lcuda link: the library must load without a GPU)
typedef int (*MemGetAddressRangeFn)(unsigned long long *, size_t *, unsigned long long);
static MemGetAddressRangeFn mem_get_address_range() {
    static MemGetAddressRangeFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (MemGetAddressRangeFn)p;
    }
    return fn;
}

}  // namespace solve
}  // namespace hcb

using namespace hcb;
using namespace hcb::solve;

extern "C" {

int hc_solve_set_formats(int force_wide_offsets, int no_x16, int no_c16) {
    g_force_wide = force_wide_offsets;
    g_no_x16 = no_x16;
    g_no_c16 = no_c16;
    return HC_OK;
}

int hc_solve_set_x8(int allow) {
    g_no_x8 = allow ? 0 : 1;
    return HC_OK;
}

int hc_mg_set_exchange(int mode) {
    HC_REQUIRE(mode >= 0 && mode <= 2, HC_ERR_INVALID, "hc_mg_set_exchange: mode %d invalid", mode);
    g_mg_exchange = mode;
    return HC_OK;
}

int hc_solve_set_l2_window(int allow) {
    g_no_l2_window = allow ? 0 : 1;
    return HC_OK;
}

int hc_solve_set_live(int mode) {
    HC_REQUIRE(mode >= -1 && mode <= 1, HC_ERR_INVALID, "hc_solve_set_live: mode %d invalid", mode);
    g_live = mode;
    return HC_OK;
}

int hc_solve_set_ell(int allow) {
    g_no_ell = allow ? 0 : 1;
    return HC_OK;
}

int hc_solve_set_small(int allow) {
    g_no_small = allow ? 0 : 1;
    return HC_OK;
}

int hc_device_info(int *h_num_sms, int *h_ctas_per_sm) {
    if (h_num_sms) *h_num_sms = num_sms();
    if (h_ctas_per_sm) *h_ctas_per_sm = occupancy();
    return HC_OK;
}

size_t hc_solve_workspace_bytes(int64_t num_nodes, int64_t num_edges) {
    const long long n = num_nodes < 0 ? 0 : num_nodes;
    return layout(n, num_edges < 0 ? 0 : num_edges, n, false).total;
}

int hc_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
             int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
             int64_t max_rec, int64_t *h_rounds, void *d_ws, size_t ws_bytes, void *stream) {
    return hc_solve_stats(d_row_offsets, d_col_indices, num_nodes, num_edges, mode, thr_count,
                          d_colors, d_rec, max_rec, h_rounds, nullptr, d_ws, ws_bytes, stream);
}

static int solve_impl(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                      int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
                      int64_t max_rec, int64_t *h_rounds, int64_t *d_stats, void *d_ws, size_t ws_bytes,
                      void *stream, bool plain);

int hc_solve_stats(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                   int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors,
                   hc_round_rec *d_rec, int64_t max_rec, int64_t *h_rounds, int64_t *d_stats,
                   void *d_ws, size_t ws_bytes, void *stream) {
    return solve_impl(d_row_offsets, d_col_indices, num_nodes, num_edges, mode, thr_count, d_colors, d_rec,
                      max_rec, h_rounds, d_stats, d_ws, ws_bytes, stream, false);
}

int hc_solve_plain(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                   int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
                   int64_t max_rec, int64_t *h_rounds, void *d_ws, size_t ws_bytes, void *stream) {
    return solve_impl(d_row_offsets, d_col_indices, num_nodes, num_edges, mode, thr_count, d_colors, d_rec,
                      max_rec, h_rounds, nullptr, d_ws, ws_bytes, stream, true);
}

// per-solve fields of Params (single GPU)
static void init_solve(Params &P, const Layout &L, char *ws, const int32_t *d_col_indices, long long n, int mode,
                       long long thr_count, int64_t *d_colors, hc_round_rec *d_rec, long long max_rec,
                       int64_t *d_stats) {
    P.ci = d_col_indices;
    P.n = n;
    P.lo = 0;
    P.nown = n;
    P.X = reinterpret_cast<unsigned *>(ws + L.x);
    P.fb0 = reinterpret_cast<unsigned *>(ws + L.fb0);
    P.fbx = reinterpret_cast<unsigned *>(ws + L.fbx);
    P.lc = reinterpret_cast<int *>(ws + L.lc);
    P.lcnt = reinterpret_cast<int *>(ws + L.lcnt);
    P.rec = d_rec;
    P.max_rec = d_rec ? max_rec : 0;
    P.colors_out = reinterpret_cast<long long *>(d_colors);
    P.mode = mode;
    P.thr = thr_count;
    P.stats = reinterpret_cast<long long *>(d_stats);
}

// the kernel choice from the preprocessing verdicts (hc_solve: x16 may be
// speculative; a plan keeps 16-bit words only where they are exact)
struct Choice {
    bool x8, x16, x16_exact, c16, small, ell, live_ok;
};
static Choice choose(const Prep &pr, long long m) {
    Choice c;
    // 16-bit state words are exact when max degree <= 16384 (mex <= 16385;
    // no node in the hub buckets >= 16385); above that they are used
    // speculatively and the solve is redone with 32-bit words if any tentative
    // color overflows (never for the BASELINE graphs)
    c.x16_exact = pr.tot[9] + pr.tot[10] + pr.tot[11] + pr.tot[12] == 0;
    c.x16 = (HC_FMT16 != 0) && !g_no_x16;
    c.c16 = pr.c16_ok;
    // bin-0-only graphs (every degree <= 16) run the SMALL kernel
    c.small = !g_no_small;
    for (int k = 1; k < NKEY; ++k) c.small = c.small && pr.tot[k] == 0;
    // 8-bit state words (colors <= 127) when every degree is <= 128 (general
    // kernel only: bin-0-only graphs measured faster with 16 bits): exact up
    // to degree 126 (mex <= deg + 1); a tentative color above 127 (two
    // degrees only) flags the overflow and the solve is redone with 16 bits.
    // ER-2^25: the 33.5 MB state array stays L2-resident (16-bit: 67 MB)
    bool upto128 = true;
    for (int k = 3; k < NKEY; ++k) upto128 = upto128 && (k == 8 || pr.tot[k] == 0);
    c.x8 = c.x16 && !g_no_x8 && upto128 && !c.small;
    c.ell = pr.ell_ok;
    // live lower lists pay on skewed graphs large enough to be bandwidth-bound
    // (RMAT-26 601 -> 435 ms, RMAT-22 31.4 -> 28.7 ms); ER-2^25 (no hubs) and
    // RMAT-16 (latency-bound) measured slower with them
    unsigned long long hubs = 0;
    for (int k = 9; k < NKEY; ++k) hubs += pr.tot[k];
    c.live_ok = g_live >= 0 ? g_live != 0 : (hubs > 0 && m >= (1LL << 25));
    return c;
}
// (pure topology sweeps read the static rows and measured faster without live lists)
static bool live_for(const Choice &c, int mode) { return c.live_ok && (g_live == 1 || mode != HC_MODE_TOPO); }

// the forbidden-color extension words (fb0 is zeroed by the kernel) and the
// live-list counts (-1: not scanned yet) of a solve
static cudaError_t reset_solve_buffers(const Params &P, const Layout &L, long long n, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(P.fbx, 0, L.fbx_bytes, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(P.lcnt, 0xff, 4 * (size_t)n, st);
    return e;
}

// stream-ordered reset of the per-solve state and the cooperative launch
// (no host synchronisation); info_dst: where the (rounds, record overflow /
// stall, format overflow) triple is copied (host for hc_solve, device for
// hc_solve_launch)
static int launch_solve(Params &P, const Layout &L, const unsigned long long *d_totals, long long n, bool narrow,
                        bool x16, bool c16, bool small, bool ell, bool live, bool plain, int64_t *d_stats,
                        void *info_dst, cudaMemcpyKind info_kind, cudaStream_t st, bool x8 = false,
                        bool fresh = false) {
    // fresh: hc_solve's first launch -- prepare() has just reset the control
    // block and the hub slots and copied the totals, and the bitmap / live
    // count resets were queued before its sync (reset_solve_buffers), so
    // nothing but the launch is issued after the host sync
    if (!fresh) {
        HC_CUDA_TRY(cudaMemsetAsync(P.ctrl, 0, offsetof(Ctrl, segcnt), st));
        copy_totals_kernel<<<1, 32, 0, st>>>(d_totals, P.ctrl);
        HC_CHECK_LAUNCH();
        HC_CUDA_TRY(cudaMemsetAsync(P.hub_acc, 0, sizeof(HubAcc) * MAX_SPLIT_SLOTS, st));
        HC_CUDA_TRY(reset_solve_buffers(P, L, n, st));
    }
    if (d_stats && P.max_rec)
        HC_CUDA_TRY(cudaMemsetAsync(d_stats, 0, sizeof(int64_t) * 2 * (size_t)P.max_rec, st));
    void *args[] = {&P};
    x8 = x8 && narrow && d_stats == nullptr && !live && !small;  // (the instantiations select_kernel has)
    const void *fn = select_kernel(narrow, x16, c16, d_stats != nullptr, small, plain, ell, live, x8);
    const size_t xbytes = (size_t)n * (x8 ? 1 : x16 && narrow ? 2 : 4);
    const int per_sm = occupancy_of(fn);
    HC_REQUIRE(per_sm > 0, HC_ERR_CUDA, "hc_solve: occupancy query failed");
    P.nblocks = (unsigned)(per_sm * std::max(1, num_sms()));
    bool windowed = false;
    // the L2 window pays on bin-0-only graphs (grid4096: 464 -> 443 ms); with
    // 8-bit words ER-2^25's 33.5 MB array would qualify too, but measured
    // 46.6 -> 50.1 ms with it (its gathers already hit; the set-aside shrinks
    // the L2 left to the column and list streams)
    HC_CUDA_TRY(launch_persistent(fn, P.nblocks, args, st, P.X, small ? xbytes : 0, true, &windowed));
    // the persisting lines go back to normal: nothing of this solve stays
    // pinned in L2 for the caller's next kernel (or the next solve)
    if (windowed) HC_CUDA_TRY(l2_demote(P.X, xbytes, st));
    HC_CUDA_TRY(cudaMemcpyAsync(info_dst, &P.ctrl->rounds, 3 * sizeof(long long), info_kind, st));
    return HC_OK;
}

static int solve_impl(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                      int64_t num_edges, int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec,
                      int64_t max_rec, int64_t *h_rounds, int64_t *d_stats, void *d_ws, size_t ws_bytes,
                      void *stream, bool plain) {
    HC_REQUIRE(num_nodes >= 0 && num_nodes < 0x7fffffffLL, HC_ERR_INVALID,
               "hc_solve: num_nodes %lld out of range", (long long)num_nodes);
    HC_REQUIRE(num_edges >= 0, HC_ERR_INVALID, "hc_solve: num_edges < 0");
    HC_REQUIRE(mode >= HC_MODE_DATA && mode <= HC_MODE_HYBRID, HC_ERR_INVALID,
               "hc_solve: mode %d invalid", mode);
    HC_REQUIRE(max_rec >= 0, HC_ERR_INVALID, "hc_solve: max_rec < 0");
    cudaStream_t st = as_stream(stream);
    if (h_rounds) *h_rounds = 0;
    if (num_nodes == 0) return HC_OK;  // empty graph: 0 rounds (test_driver.py:88-93)
    HC_REQUIRE(d_row_offsets && d_colors && (num_edges == 0 || d_col_indices), HC_ERR_INVALID,
               "hc_solve: null pointer");
    const Layout L = layout(num_nodes, num_edges, num_nodes, false);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_solve: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P{};
    init_solve(P, L, ws, d_col_indices, num_nodes, mode, thr_count, d_colors, d_rec, max_rec, d_stats);
    Prep pr;
    HC_CUDA_TRY(reset_solve_buffers(P, L, num_nodes, st));  // (queued ahead of prepare's sync)
    int rc = prepare(P, L, ws, d_row_offsets, num_nodes, num_edges, false, pr, st,
                     reinterpret_cast<unsigned long long *>(ws + L.ell));
    if (rc != HC_OK) return rc;
    const Choice ch = choose(pr, num_edges);
    bool x16 = ch.x16, x8 = ch.x8, fresh = true;
    long long info[3];
    for (;;) {
        rc = launch_solve(P, L, pr.d_totals, num_nodes, pr.narrow, x16, ch.c16, ch.small, ch.ell, live_for(ch, mode),
                          plain, d_stats, info, cudaMemcpyDeviceToHost, st, x8, fresh);
        fresh = false;  // a rerun resets everything again
        if (rc != HC_OK) return rc;
        HC_CUDA_TRY(cudaStreamSynchronize(st));
        const unsigned overflow = (unsigned)(info[2] & 0xffffffffLL);
        if (x8 && overflow && pr.narrow && !d_stats && !live_for(ch, mode) && !ch.small) {
            x8 = false;  // redo with 16-bit state words
            continue;
        }
        if (!(x16 && overflow) || ch.x16_exact) break;
        x16 = false;  // redo with 32-bit state words
    }
    if (h_rounds) *h_rounds = info[0];
    HC_REQUIRE(info[1] != 2, HC_ERR_STALLED, "hc_solve: no convergence after %lld rounds (internal error)", info[0]);
    HC_REQUIRE(!info[1], HC_ERR_RECORDS, "hc_solve: %lld rounds exceed the %lld-record buffer",
               info[0], (long long)max_rec);
    return HC_OK;
}

int hc_solve_plan_graph(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                        int64_t num_edges, void *d_ws, size_t ws_bytes, hc_solve_plan *h_plan, void *stream) {
    HC_REQUIRE(h_plan, HC_ERR_INVALID, "hc_solve_plan_graph: null plan");
    HC_REQUIRE(num_nodes >= 0 && num_nodes < 0x7fffffffLL, HC_ERR_INVALID,
               "hc_solve_plan_graph: num_nodes %lld out of range", (long long)num_nodes);
    HC_REQUIRE(num_edges >= 0, HC_ERR_INVALID, "hc_solve_plan_graph: num_edges < 0");
    memset(h_plan, 0, sizeof *h_plan);
    h_plan->num_nodes = num_nodes;
    h_plan->num_edges = num_edges;
    if (num_nodes == 0) return HC_OK;
    HC_REQUIRE(d_row_offsets && (num_edges == 0 || d_col_indices), HC_ERR_INVALID, "hc_solve_plan_graph: null pointer");
    const Layout L = layout(num_nodes, num_edges, num_nodes, false);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_solve_plan_graph: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    cudaStream_t st = as_stream(stream);
    Params P{};
    init_solve(P, L, ws, d_col_indices, num_nodes, HC_MODE_HYBRID, 0, nullptr, nullptr, 0, nullptr);
    Prep pr;
    const int rc = prepare(P, L, ws, d_row_offsets, num_nodes, num_edges, false, pr, st,
                           reinterpret_cast<unsigned long long *>(ws + L.ell));
    if (rc != HC_OK) return rc;
    const Choice ch = choose(pr, num_edges);
    h_plan->narrow = pr.narrow;
    h_plan->x16 = ch.x16 && ch.x16_exact;  // a launch never redoes the solve
    h_plan->c16 = ch.c16;
    h_plan->small = ch.small;
    h_plan->ell = ch.ell;
    h_plan->live = ch.live_ok;
    h_plan->totals_offset = (int64_t)(reinterpret_cast<char *>(pr.d_totals) - ws);
    return HC_OK;
}

int hc_solve_launch(const hc_solve_plan *h_plan, const int64_t *d_row_offsets, const int32_t *d_col_indices,
                    int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                    int64_t *d_info, void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(h_plan && d_info, HC_ERR_INVALID, "hc_solve_launch: null plan / info");
    HC_REQUIRE(mode >= HC_MODE_DATA && mode <= HC_MODE_HYBRID, HC_ERR_INVALID, "hc_solve_launch: mode %d invalid", mode);
    HC_REQUIRE(max_rec >= 0, HC_ERR_INVALID, "hc_solve_launch: max_rec < 0");
    cudaStream_t st = as_stream(stream);
    const long long n = h_plan->num_nodes, m = h_plan->num_edges;
    if (n == 0) {
        HC_CUDA_TRY(cudaMemsetAsync(d_info, 0, 3 * sizeof(int64_t), st));
        return HC_OK;
    }
    HC_REQUIRE(d_row_offsets && d_colors && (m == 0 || d_col_indices), HC_ERR_INVALID, "hc_solve_launch: null pointer");
    const Layout L = layout(n, m, n, false);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_solve_launch: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P{};
    init_solve(P, L, ws, d_col_indices, n, mode, thr_count, d_colors, d_rec, max_rec, nullptr);
    bind_params(P, L, ws, d_row_offsets, h_plan->narrow != 0);
    P.ell = reinterpret_cast<const unsigned long long *>(ws + L.ell);
    Choice ch{};
    ch.live_ok = h_plan->live != 0;
    return launch_solve(P, L, reinterpret_cast<const unsigned long long *>(ws + h_plan->totals_offset), n,
                        h_plan->narrow != 0, h_plan->x16 != 0, h_plan->c16 != 0, h_plan->small != 0,
                        h_plan->ell != 0, live_for(ch, mode), false, nullptr, d_info, cudaMemcpyDeviceToDevice, st);
}

/* ---------------------------------------------------------------- multi-GPU */

size_t hc_mg_shared_bytes(int64_t num_nodes) {
    return mg_x_bytes(num_nodes < 0 ? 0 : num_nodes) + align_up(sizeof(Mbox), 256);
}

size_t hc_mg_workspace_bytes(int64_t num_nodes, int64_t num_edges, int64_t lo, int64_t hi) {
    // num_edges: the shard's half-edges
    const long long n = num_nodes < 0 ? 0 : num_nodes;
    const long long nown = hi > lo ? hi - lo : 0;
    return layout(n, num_edges < 0 ? 0 : num_edges, nown, true).total;
}

int hc_mg_alloc_shared(size_t bytes, void **h_dptr) {
    HC_REQUIRE(h_dptr && bytes > 0, HC_ERR_INVALID, "hc_mg_alloc_shared: bad arguments");
    void *p = nullptr;
    HC_CUDA_TRY(cudaMalloc(&p, bytes));
    const cudaError_t e = cudaMemset(p, 0, bytes);
    if (e != cudaSuccess) {
        cudaFree(p);
        HC_CUDA_TRY(e);
    }
    *h_dptr = p;
    return HC_OK;
}

int hc_mg_free_shared(void *d_ptr) {
    if (d_ptr) HC_CUDA_TRY(cudaFree(d_ptr));
    return HC_OK;
}

int hc_mg_ipc_export(const void *d_ptr, void *h_handle, int64_t *h_offset) {
    HC_REQUIRE(d_ptr && h_handle && h_offset, HC_ERR_INVALID, "hc_mg_ipc_export: null pointer");
    MemGetAddressRangeFn range = mem_get_address_range();
    HC_REQUIRE(range, HC_ERR_CUDA, "hc_mg_ipc_export: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    HC_REQUIRE(range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) == 0, HC_ERR_CUDA,
               "hc_mg_ipc_export: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    HC_CUDA_TRY(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
    static_assert(sizeof(cudaIpcMemHandle_t) == HC_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(h_handle, &h, sizeof h);
    *h_offset = (int64_t)((uintptr_t)d_ptr - (uintptr_t)base);
    return HC_OK;
}

int hc_mg_ipc_import(const void *h_handle, int64_t offset, void **h_dptr) {
    HC_REQUIRE(h_handle && h_dptr && offset >= 0, HC_ERR_INVALID, "hc_mg_ipc_import: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handle, sizeof h);
    void *base = nullptr;
    HC_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *h_dptr = (char *)base + offset;
    return HC_OK;
}

int hc_mg_ipc_close(void *d_ptr, int64_t offset) {
    HC_REQUIRE(d_ptr && offset >= 0, HC_ERR_INVALID, "hc_mg_ipc_close: bad arguments");
    HC_CUDA_TRY(cudaIpcCloseMemHandle((char *)d_ptr - offset));
    return HC_OK;
}

int hc_mg_prepare(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                  int64_t num_edges, const int64_t *h_bounds, int rank, int world, void *const *h_shared,
                  int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                  int ctas, int64_t timeout_ms, int64_t global_max_degree, void *d_ws, size_t ws_bytes,
                  void *stream) {
    HC_REQUIRE(h_bounds && world >= 1 && world <= MG_MAX_WORLD && rank >= 0 && rank < world, HC_ERR_INVALID,
               "hc_mg_solve: rank %d / world %d invalid (world <= %d)", rank, world, MG_MAX_WORLD);
    for (int q = 0; q < world; ++q)
        HC_REQUIRE(h_bounds[q] <= h_bounds[q + 1], HC_ERR_INVALID, "hc_mg_solve: bounds not ascending");
    HC_REQUIRE(h_bounds[0] == 0 && h_bounds[world] == num_nodes, HC_ERR_INVALID,
               "hc_mg_solve: bounds must cover [0, num_nodes)");
    const int64_t lo = h_bounds[rank], hi = h_bounds[rank + 1];
    HC_REQUIRE(num_nodes >= 1 && num_nodes < 0x7fffffffLL, HC_ERR_INVALID,
               "hc_mg_solve: num_nodes %lld out of range", (long long)num_nodes);
    HC_REQUIRE(num_edges >= 0, HC_ERR_INVALID, "hc_mg_solve: num_edges < 0");
    HC_REQUIRE(world >= 1 && world <= MG_MAX_WORLD && rank >= 0 && rank < world, HC_ERR_INVALID,
               "hc_mg_solve: rank %d / world %d invalid (world <= %d)", rank, world, MG_MAX_WORLD);
    HC_REQUIRE(lo >= 0 && hi >= lo && hi <= num_nodes, HC_ERR_INVALID, "hc_mg_solve: bad owned range");
    HC_REQUIRE(mode >= HC_MODE_DATA && mode <= HC_MODE_HYBRID, HC_ERR_INVALID,
               "hc_mg_solve: mode %d invalid", mode);
    HC_REQUIRE(max_rec >= 0 && ctas >= 0, HC_ERR_INVALID, "hc_mg_solve: bad max_rec / ctas");
    HC_REQUIRE(d_row_offsets && (num_edges == 0 || d_col_indices) && h_shared &&
                   (hi == lo || d_colors), HC_ERR_INVALID, "hc_mg_solve: null pointer");
    for (int q = 0; q < world; ++q) HC_REQUIRE(h_shared[q], HC_ERR_INVALID, "hc_mg_solve: null shared[%d]", q);
    cudaStream_t st = as_stream(stream);
    const Layout L = layout(num_nodes, num_edges, hi - lo, true);
    HC_REQUIRE(d_ws && ws_bytes >= L.total, HC_ERR_WORKSPACE,
               "hc_mg_solve: workspace %zu bytes < required %zu", ws_bytes, L.total);
    char *ws = reinterpret_cast<char *>(d_ws);
    Params P{};
    P.ci = d_col_indices;
    P.n = num_nodes;
    P.lo = lo;
    P.nown = hi - lo;
    P.rec = d_rec;
    P.max_rec = d_rec ? max_rec : 0;
    P.colors_out = reinterpret_cast<long long *>(d_colors);
    P.mode = mode;
    P.thr = thr_count;
    P.rank = rank;
    P.world = world;
    P.timeout_ns = (timeout_ms > 0 ? timeout_ms : 60000) * 1000000LL;
    P.exchange = g_mg_exchange;
    HC_REQUIRE(global_max_degree >= 0 || world == 1, HC_ERR_INVALID,
               "hc_mg_solve: global_max_degree required when world > 1");
    Prep pr;
    int rc = prepare(P, L, ws, d_row_offsets, num_nodes, num_edges, global_max_degree < 0, pr, st);
    if (rc != HC_OK) return rc;
    if (global_max_degree >= 0) pr.max_degree = (unsigned long long)global_max_degree;
    // peer masks of the owned nodes + boundary zones
    unsigned char *bnd = reinterpret_cast<unsigned char *>(ws + L.bnd);
    long long *d_bounds = reinterpret_cast<long long *>(ws + L.ptrs + 2 * sizeof(void *) * MG_MAX_WORLD);
    unsigned long long *d_zones = reinterpret_cast<unsigned long long *>(d_bounds + MG_MAX_WORLD + 1);
    long long hb[MG_MAX_WORLD + 1] = {};
    for (int q = 0; q <= world; ++q) hb[q] = h_bounds[q];
    HC_CUDA_TRY(cudaMemcpyAsync(d_bounds, hb, sizeof hb, cudaMemcpyHostToDevice, st));
    HC_CUDA_TRY(cudaMemsetAsync(d_zones, 0, 24, st));
    if (hi > lo && num_edges > 0) {
        const long long blocks = std::min<long long>((hi - lo + 7) / 8, (long long)std::max(1, num_sms()) * 16);
        mg_boundary_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const long long *>(d_row_offsets) - lo,
                                                              d_col_indices, d_bounds, world, rank, bnd, d_zones);
        HC_CHECK_LAUNCH();
    }
    unsigned long long hz[3] = {0, 0, 0};
    HC_CUDA_TRY(cudaMemcpyAsync(hz, d_zones, sizeof hz, cudaMemcpyDeviceToHost, st));
    P.bnd = bnd - lo;
    // peer tables: every rank's replica and mailbox (pointers valid in this process)
    void *tab[2 * MG_MAX_WORLD] = {};
    for (int q = 0; q < world; ++q) {
        tab[q] = h_shared[q];
        tab[MG_MAX_WORLD + q] = (char *)h_shared[q] + mg_x_bytes(num_nodes);
    }
    void **d_tab = reinterpret_cast<void **>(ws + L.ptrs);
    HC_CUDA_TRY(cudaMemcpyAsync(d_tab, tab, sizeof tab, cudaMemcpyHostToDevice, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    P.zlo = (long long)hz[0];
    P.zhi = (long long)hz[1];
    P.peer_words = (long long)hz[2];
    P.peer_x = d_tab;
    P.peer_mbox = reinterpret_cast<Mbox *const *>(d_tab + MG_MAX_WORLD);
    P.X = h_shared[rank];
    P.mbox = reinterpret_cast<Mbox *>(tab[MG_MAX_WORLD + rank]);
    // every rank must pick the same state-word width: decided on the whole graph
    const bool x16 = (HC_FMT16 != 0) && !g_no_x16 && pr.max_degree <= 16384ull;
    // the kernel family is a whole-graph decision too: ranks sharing one GPU
    // (tests) must run kernels with the same shared-memory footprint to
    // co-reside (an SM's carve-out cannot change while a CTA lives on it)
    const bool small = !g_no_small && pr.max_degree <= 16ull;
    const void *fn = select_kernel_mg(pr.narrow, x16, pr.c16_ok, small);
    const int per_sm = occupancy_of(fn);
    HC_REQUIRE(per_sm > 0, HC_ERR_CUDA, "hc_mg_solve: occupancy query failed");
    const unsigned full = (unsigned)(per_sm * std::max(1, num_sms()));
    P.nblocks = ctas > 0 ? std::min((unsigned)ctas, full) : full;
    std::lock_guard<std::mutex> lk(g_mg_mu);
    g_mg_prepared[d_ws] = MgLaunch{P, fn, ctas > 0};
    return HC_OK;
}

int hc_mg_launch(void *d_ws, void *stream) {
    MgLaunch L;
    {
        std::lock_guard<std::mutex> lk(g_mg_mu);
        auto it = g_mg_prepared.find(d_ws);
        HC_REQUIRE(it != g_mg_prepared.end(), HC_ERR_INVALID, "hc_mg_launch: workspace not prepared");
        L = it->second;
    }
    cudaStream_t st = as_stream(stream);
    void *args[] = {&L.P};
    if (L.regular)  // caller-sized grid (several ranks sharing one GPU): regular launch
        HC_CUDA_TRY(cudaLaunchKernel(L.fn, dim3(L.P.nblocks), dim3(BLOCK), args, 0, st));
    else
        HC_CUDA_TRY(cudaLaunchCooperativeKernel(L.fn, dim3(L.P.nblocks), dim3(BLOCK), args, 0, st));
    return HC_OK;  // asynchronous: hc_mg_wait collects the outcome
}

int hc_mg_solve(const int64_t *d_row_offsets, const int32_t *d_col_indices, int64_t num_nodes,
                int64_t num_edges, const int64_t *h_bounds, int rank, int world, void *const *h_shared,
                int mode, int64_t thr_count, int64_t *d_colors, hc_round_rec *d_rec, int64_t max_rec,
                int ctas, int64_t timeout_ms, int64_t global_max_degree, void *d_ws, size_t ws_bytes,
                void *stream) {
    const int rc = hc_mg_prepare(d_row_offsets, d_col_indices, num_nodes, num_edges, h_bounds, rank, world,
                                 h_shared, mode, thr_count, d_colors, d_rec, max_rec, ctas, timeout_ms,
                                 global_max_degree, d_ws, ws_bytes, stream);
    return rc != HC_OK ? rc : hc_mg_launch(d_ws, stream);
}

int hc_mg_wait(void *d_ws, int64_t *h_rounds, void *stream) {
    HC_REQUIRE(d_ws, HC_ERR_INVALID, "hc_mg_wait: null workspace");
    cudaStream_t st = as_stream(stream);
    const Ctrl *C = reinterpret_cast<const Ctrl *>(d_ws);  // the control block leads the layout
    struct {
        long long rounds, rec_overflow;
    } info;
    unsigned abort = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&info, &C->rounds, sizeof info, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaMemcpyAsync(&abort, &C->abort, sizeof abort, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    HC_REQUIRE(!abort, HC_ERR_TIMEOUT,
               "hc_mg_solve: a peer did not reach a cross-GPU barrier in time (this rank in round %lld)",
               info.rounds);
    if (h_rounds) *h_rounds = info.rounds;
    HC_REQUIRE(!info.rec_overflow, HC_ERR_RECORDS, "hc_mg_solve: %lld rounds exceed the record buffer",
               info.rounds);
    return HC_OK;
}

}  // extern "C"
