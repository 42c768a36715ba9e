// hcb_solve_dev.cuh -- the device side of hc_solve: state encoding, bins,
// worklists, assign / resolve tiles and the persistent solve_kernel template.
// Included by hcb_solve.cu (host side: preprocessing, launch, C-ABI) and by
// hcb_solve_inst.cu, which instantiates the solve_kernel variants in
// separate translation units (HC_INST_GROUP) so they compile in parallel.
#pragma once
// device-resident IPGC solve (hc_solve).
//
// Replaces the reference's whole `color_graph` round loop
// (pkg/src/hybridcolor/driver.py:122-176) together with the round functions
// (coloring.py:113-176), the kernels (_kernels.pyx:29-149) and the worklist
// swap (worklist.py:77-91) by ONE cooperatively launched persistent kernel
// (three 512-thread CTAs per SM): every round is
//     assign -> grid barrier -> resolve -> grid barrier
// with the hybrid mode decision, the worklist and the per-round records kept
// on the device, so there is no host round trip per round.
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
// Work distribution (IrGL-style nested parallelism).
// Nodes are binned once by degree; each bin has its own granularity:
//   bin 0  deg <= 16        one thread per node, NPT=2 nodes per thread with
//                           all their loads batched (memory-level parallelism)
//   bin 1  17..32           a group of 8 lanes per node (4 nodes per warp)
//   bin 2  33..64           16 lanes per node (2 per warp)
//   bin 3  65..4096         one warp per node; one CTA per node in rounds with
//                           few active bin-3 nodes (latency regime)
//   bin 4  > 4096 (hubs)    one CTA per node
// Within a group every lane issues 4 neighbour loads before consuming any.
// The mex is first taken over a 64-bit register mask of colors 1..64 (OR-
// reduced across the group); only nodes whose colors 1..64 are all taken fall
// back to a shared-memory bitmap window.
// The always-maintained worklist is kept per bin and double buffered.  Each
// phase hands out units with ONE atomic per unit: hubs first (largest work
// first), then chunks of bins 3, 2, 1, 0.  Losers of chunk c are compacted
// into output segment c of the next worklist (order-preserving for bin 0) and
// the chunk writes its loser count; the next round rebuilds the segment prefix
// in shared memory.  So pushes need no global atomics, the worklist stays
// (nearly) sorted by id, and topology-driven rounds (static bin lists +
// activity test) and data-driven rounds (segmented dynamic lists) share the
// same code.
//
// Row offsets are read as int32 when num_edges < 2^31 (a copy made in the
// preprocessing), halving the offset traffic; int64 otherwise.  Column loads
// are streaming (evict-first) so the X gathers keep L2.
#include <string.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "hcb_partition.cuh"

namespace hcb {
namespace solve {

#ifndef HC_BLOCK
#define HC_BLOCK 512
#endif
#ifndef HC_NPT
#define HC_NPT 2
#endif
constexpr int BLOCK = HC_BLOCK;
#ifndef HC_FMT16
#define HC_FMT16 1
#endif
#ifndef HC_MINB
#define HC_MINB 3   // 3 x 512-thread CTAs per SM (42 registers): ER-2^25 108 -> 95 ms, RMAT-26 1624 -> 1544 ms
#endif
constexpr int MIN_CTAS = HC_MINB;        // resident CTAs per SM the register budget targets
#ifndef HC_MINB_SMALL
#define HC_MINB_SMALL 3
#endif
constexpr int MIN_CTAS_SMALL = HC_MINB_SMALL;  // the same for bin-0-only graphs (SmemT<true>)
constexpr int NW = BLOCK / 32;
constexpr int NPT = HC_NPT;              // bin-0 nodes per thread per tile
#ifndef HC_MG_PLAIN_BARRIER
#define HC_MG_PLAIN_BARRIER 0
#endif
#ifndef HC_PHASE_TIMES
#define HC_PHASE_TIMES 0
#endif
#ifndef HC_LIVE_GROUPS
#define HC_LIVE_GROUPS 0   // live lists also for bins 1-2 (8- and 16-lane groups): half the spills without (RMAT-26 422.5 -> 420.5 ms)
#endif
#ifndef HC_LIVE
#define HC_LIVE 1   // resolve scans of bins 1..4 compact each node's lower list to its uncolored entries
#endif
#ifndef HC_GROUP_PREFETCH
#define HC_GROUP_PREFETCH 1   // resolve: group tiles fetch the next tile's entries one tile ahead
#endif
#ifndef HC_PAIR
#define HC_PAIR 2   // bin-0-only kernel: tiles per loser-compaction barrier
#endif
#ifndef HC_NPT_SMALL
#define HC_NPT_SMALL 2
#endif
constexpr int NPT_SMALL = HC_NPT_SMALL;  // the same in the bin-0-only kernel (more CTAs, fewer registers)
constexpr int NPT_MAX = NPT > NPT_SMALL ? NPT : NPT_SMALL;  // sizes the shared tables
// bitmap assign (phase 0 with forbidden-color bitmaps): nodes per thread per
// tile.  The phase is a pure stream over the lists (entry, activity word,
// bitmap word -> tentative word), so every bin but the hubs runs thread per
// node and a thread keeps NPA independent nodes in flight.
#ifndef HC_NPA
#define HC_NPA 4
#endif
#ifndef HC_NPA_SMALL
#define HC_NPA_SMALL 8
#endif
constexpr int NSEG_BINS = 4;             // bins 0..3 are segmented; bin 4 (hubs) is dense
constexpr int BIN_HUB = 4;
constexpr int NBIN = 5;
constexpr int HUB_MIN = 4097;            // deg >= HUB_MIN -> hub
#ifndef HC_HUB_U
#define HC_HUB_U 4
#endif
constexpr int HU = HC_HUB_U;             // column loads in flight per thread in the CTA-per-node paths
constexpr int HUB_WORDS = 512;           // CTA bitmap window: 16384 colors per pass
constexpr int WIN_WORDS = 32;            // warp bitmap window: 1024 colors per pass
#ifndef HC_MAXSEG
#define HC_MAXSEG 2048
#endif
constexpr int MAXSEG = HC_MAXSEG;        // output segments per bin per round
static_assert(MAXSEG % BLOCK == 0, "prefix scan: whole items per thread");
constexpr unsigned FBIT = 0x80000000u;
constexpr unsigned CMASK = 0x7fffffffu;

__host__ __device__ constexpr int bin_of_degree(long long d) {
    return d <= 16 ? 0 : d <= 32 ? 1 : d <= 64 ? 2 : d < HUB_MIN ? 3 : 4;
}

constexpr int MAX_PEND = 1024;
#ifndef HC_DEFER_PUSH
#define HC_DEFER_PUSH 1   // winning hubs' pushes split across every CTA at the next round start
#endif
#ifndef HC_DEFER_MIN
#define HC_DEFER_MIN 65536   // ... for hubs of at least this degree
#endif
struct Ctrl {
    GridBarrier bar;
    int error;
    int pad0;
    unsigned long long nstat[NBIN];              // static bin sizes
    unsigned long long hub_cnt[2];               // hub worklist size per parity
    unsigned long long conflicts[2];
    unsigned int unit_ctr[2][2];                 // [phase][parity]
    long long rounds_live;  // current round (development timing builds)
    long long rounds;       // (rounds, rec_overflow, fmt_overflow) are read back as one triple
    long long rec_overflow;
    unsigned fmt_overflow;                       // a tentative color exceeded the state word
    unsigned pad1;
    // multi-GPU: this rank's next-worklist size per parity, the global sums of
    // the last round (|W'|, conflicts) and the abort flag of a timed-out barrier
    unsigned long long wl_next[2];
    unsigned long long g_wl, g_conf;
    unsigned abort;
    unsigned pad2;
    unsigned long long plain_cnt[2][NSEG_BINS];  // Plain variant: dense list sizes per parity and bin
    // winning hubs of a round whose bitmap pushes all CTAs share at the start
    // of the next round (pend_cnt is reset after that; entries past MAX_PEND
    // are pushed inline by their CTA)
    unsigned pend_cnt[2];
    unsigned segcnt[2][NSEG_BINS][MAXSEG];       // [parity][bin][segment] loser counts
    int pend[2][MAX_PEND];
};

// Multi-GPU mailbox, one per rank, in the rank's peer-mapped shared region
// (after its state-word replica).  Rank r's cross-GPU barrier number e writes
// three tagged words (e_lo32 << 32 | value32: |W'|, conflicts lo / hi) into
// slot [e & 1][r] of every rank's mailbox and waits until every slot
// [e & 1][*] of its own mailbox carries tag e.  Tagged words make each word
// self-validating, so the post is ONE system fence + relaxed stores and the
// wait is relaxed polls + ONE fence (no per-word release / acquire).  Two slot
// sets suffice: a rank can post e+2 only after every rank posted e+1, i.e.
// after every rank finished reading the payloads of e.
constexpr int MG_MAX_WORLD = 8;
struct MboxSlot {
    unsigned long long w[3];
    unsigned long long pad;
};
struct Mbox {
    MboxSlot slot[2][MG_MAX_WORLD];
    unsigned long long last_epoch;  // barriers used by the previous solves (all ranks agree)
    unsigned long long pad[3];
};

// per-hub merge slot for hubs split across several CTAs (latency regime)
constexpr int HA_WORDS = 62;                   // colors 65..2048 beyond the 64-bit mask
#ifndef HC_UPC3
#define HC_UPC3 16   // bin-3 work units per CTA (at least one warp tile each)
#endif
#ifndef HC_BIN3_CTA
#define HC_BIN3_CTA 0   // every bin-3 node CTA per node when at most 2 x #CTAs are active (RMAT-16 2.66 vs 2.32 ms without)
#endif
#ifndef HC_K3
#define HC_K3 100  // leading bin-3 nodes taken CTA per node, in percent of the CTAs
#endif
#ifndef HC_MAX_SPLIT
#define HC_MAX_SPLIT 1024
#endif
#ifndef HC_NO_SPLIT
#define HC_NO_SPLIT 0   // experiments: never split hubs into slices
#endif
#ifndef HC_SPLIT_ANY
#define HC_SPLIT_ANY 0   // split the active hubs whenever they fit the slots (not only when fewer than the CTAs)
#endif
constexpr int MAX_SPLIT_SLOTS = HC_MAX_SPLIT;
struct HubAcc {
    unsigned long long mask;                   // colors 1..64 seen (assign)
    unsigned words[HA_WORDS];                  // colors 65..2048 seen (assign)
    unsigned cnt, low;                         // conflicts / lower neighbours (resolve)
    unsigned arrive;                           // slices done
    unsigned pad;
};

struct Params {
    const void *ro;            // int32 or int64 row offsets (template OffT)
    const int *ci;
    const short *ci16;         // delta-encoded columns (Fmt CT = short)
    // ELL4 rows (Fmt ELL): per node 4 int16 deltas v-u in one 8-byte word,
    // row order, 0-padded -- every degree <= 4 and |v-u| < 2^15
    const unsigned long long *ell;
    long long n;
    void *X;                   // state words (Fmt XT)
    int *stat;                 // static lists, bins contiguous
    int *dyn[2][NBIN];         // dynamic lists per parity and bin
    // (row offset << 16 | degree) of every list entry of bins 0-3, so a list
    // read yields the adjacency range without a dependent row-offset load
    unsigned long long *stat_od;
    unsigned long long *dyn_od[2][NSEG_BINS];
    Ctrl *ctrl;
    hc_round_rec *rec;
    long long max_rec;
    long long *colors_out;
    int mode;
    long long thr;
    unsigned nblocks;
    long long *stats;          // optional int64[max_rec][2]: (assign edges, resolve lower edges)
    HubAcc *hub_acc;           // MAX_SPLIT_SLOTS merge slots (zeroed; reset by their last slice)
    unsigned *fmt_overflow;    // set when a tentative color does not fit the state word
    // forbidden-color bitmaps (single GPU): fb0[u] bit c-1 = a committed
    // neighbour of u has color c (c <= 32); colors 33..deg(u)+1 in
    // fbx[(ro[u] >> 5) + (c - 33) / 32].  Winners set the bits of their color
    // in every neighbour once, when they commit; assign is then the mex of the
    // node's own bitmap instead of a scan of its adjacency.
    unsigned *fb0;
    unsigned *fbx;
    // live lower lists (single GPU, bins 1..4): once u has been scanned in a
    // data-driven round, its lower neighbours that were still uncolored then
    // are lc[ro[u] .. ro[u] + live) (any order).  Resolve counts conflicts
    // only against uncolored lower neighbours (a committed one never matches:
    // T[u] avoids committed colors), and colored nodes never become
    // uncolored, so a scan may drop every committed entry for good --
    // compacted in place by the scan itself.  `live` travels in the list
    // entry's od (bins 1..3: OD_LIVE | live << 48) or in lcnt[u] (hubs; -1:
    // not scanned yet).
    int *lc;
    int *lcnt;
    long long lo, nown;        // owned node range [lo, lo + nown) (single GPU: 0, n)
    // multi-GPU (Fmt::mg) only
    const unsigned char *bnd;  // per owned node: bit q = rank q reads this word (global id index)
    long long zlo, zhi;        // boundary zones: nodes u with u - lo < zlo or hi - u <= zhi may be read by peers
    long long peer_words;      // sum over owned nodes of the peers reading them (mirror cost model)
    void *const *peer_x;       // [world] every rank's state-word replica (device array)
    Mbox *const *peer_mbox;    // [world] every rank's mailbox
    Mbox *mbox;                // this rank's mailbox
    int rank, world;
    long long timeout_ns;      // cross-GPU barrier wait limit
    int exchange;              // 0 auto (per round), 1 always mirror stores, 2 always zone copies
};

// A bin's current list: dense (static list / round 1) or segmented (the
// previous round's output: nseg segments of capacity segcap).
struct List {
    const int *base;
    const unsigned long long *od;  // per entry: row offset << 16 | degree (bins 0-3)
    unsigned long long total;
    unsigned nseg, segcap;
    bool segmented;
};

// per-round, CTA-uniform configuration kept in shared memory (registers are
// the scarce resource at 1024 threads per SM)
struct RoundCfg {
    List L[NBIN];
    const int *stat_lists[NBIN];
    const unsigned long long *stat_od[NBIN];
    unsigned long long nst[NBIN];
    unsigned csz[NSEG_BINS], nch[NSEG_BINS];  // output segment size / count per bin
    unsigned su[NSEG_BINS], nsu[NSEG_BINS];   // work-unit size / count of the group bins 1..3
    unsigned k3;                              // leading bin-3 positions processed CTA per node
    unsigned ubase[NBIN + 1];      // unit ranges: hub, bin3, bin2, bin1, bin0
    unsigned abase[NBIN + 1];      // bitmap-assign unit ranges (thread per node in every bin but the hubs)
    unsigned prev_nseg[NSEG_BINS], prev_cap[NSEG_BINS];
    unsigned hub_split;            // hubs split into equal-size edge slices (latency regime)
    unsigned hub_slice;            // edges per slice
    bool topo, ident, bin3_by_cta, ident_small;
    bool bulk;                     // multi-GPU: this round's words go to the peers by zone copies
    long long round;               // current round t (development timing builds)
};

// SMALL: the graph has only bin-0 nodes (max degree <= 16: grids, meshes,
// road networks); the kernel then carries neither the group / hub code nor
// their shared memory, so it fits more CTAs per SM with a larger L1.
template <bool SMALL>
struct SmemT {
    RoundCfg rc;
    unsigned hub_pre[SMALL ? 1 : MAX_SPLIT_SLOTS + 1];    // slice prefix over the active hubs (split rounds)
    unsigned prefix[SMALL ? 1 : NSEG_BINS][MAXSEG + 1];   // segment prefix of the current lists
    unsigned win_bm[SMALL ? 1 : NW][WIN_WORDS];
    unsigned hub_bm[SMALL ? 1 : HUB_WORDS];
    unsigned warp_tmp[NPT_MAX * NW];
    unsigned cnt_tab[2][2 * NPT_MAX * NW];
    unsigned long long red;
    int hub_first;
    unsigned unit;
    unsigned out_cnt;
    unsigned kcnt;  // live-list compaction count (resolve_cta)
    unsigned mg_abort;
};
using Smem = SmemT<false>;

// dynamic list of parity p, bin b (selects instead of a runtime-indexed
// kernel-parameter array, which would force a local-memory copy of Params)
__device__ __forceinline__ int *dyn_list(const Params &P, int p, int b) {
    return p ? P.dyn[1][b] : P.dyn[0][b];
}
__device__ __forceinline__ unsigned long long *dyn_od(const Params &P, int p, int b) {
    return p ? P.dyn_od[1][b] : P.dyn_od[0][b];
}
// od = row offset << 16 | degree (bits 16..47 and 0..15); bins 1..3 add the
// live lower count (bits 48..62) under OD_LIVE once compacted
constexpr unsigned long long OD_LIVE = 1ull << 63;
constexpr unsigned long long OD_BASE = (1ull << 48) - 1ull;
__device__ __forceinline__ long long od_off(unsigned long long od) { return (long long)((od >> 16) & 0xffffffffull); }
__device__ __forceinline__ unsigned long long od_live(unsigned long long od, unsigned kept) {
    return (od & OD_BASE) | OD_LIVE | ((unsigned long long)kept << 48);
}
__device__ __forceinline__ unsigned long long make_od(long long b, long long e) {
    return ((unsigned long long)b << 16) | (unsigned long long)(e - b);
}
// list entry loads (plain loads: __ldcg here cost the grid 5%, 608 -> 640 ms)
__device__ __forceinline__ int ld_entry(const int *p) { return *p; }
__device__ __forceinline__ unsigned long long ld_od(const unsigned long long *p) { return *p; }

__device__ __forceinline__ long long list_index(const List &L, const unsigned *prefix, unsigned long long v) {
    if (!L.segmented) return (long long)v;
    // last segment s with prefix[s] <= v (segments may be empty)
    unsigned lo = 0, hi = L.nseg;  // invariant prefix[lo] <= v < prefix[hi]
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (prefix[mid] <= v) lo = mid;
        else hi = mid;
    }
    return (long long)lo * L.segcap + (long long)(v - prefix[lo]);
}

// segment-walk variant: `s` is a segment at or before the one holding v (a
// hint carried across increasing v), advanced in place
__device__ __forceinline__ long long list_index_walk(const List &L, const unsigned *prefix,
                                                     unsigned long long v, unsigned &s) {
    if (!L.segmented) return (long long)v;
    while (prefix[s + 1] <= v) ++s;
    return (long long)s * L.segcap + (long long)(v - prefix[s]);
}

// segment holding v (binary search; v < total)
__device__ __forceinline__ unsigned list_segment(const List &L, const unsigned *prefix, unsigned long long v) {
    if (!L.segmented) return 0;
    unsigned lo = 0, hi = L.nseg;
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        if (prefix[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// chunk size so a bin produces at most MAXSEG segments; multiple of `tile`
__device__ __forceinline__ unsigned chunk_size(unsigned long long total, unsigned tile) {
    unsigned long long c = (total + MAXSEG - 1) / MAXSEG;
    c = (c + tile - 1) / tile * tile;
    return (unsigned)max(c, (unsigned long long)tile);
}

__device__ __forceinline__ void mark(unsigned *bm, unsigned c) {
    atomicOr(&bm[(c - 1u) >> 5], 1u << ((c - 1u) & 31u));
}

// loser count of output segment c of bin `bin`; the multi-GPU solve also
// keeps this rank's next-worklist total for the cross-GPU reduction
// (thread 0 of the CTA; the multi-GPU total is kept per CTA and added once
// per round at the end of resolve)
__shared__ unsigned long long s_wl_acc;
template <bool MG>
__device__ __forceinline__ void seg_put(const Params &P, int np, int bin, unsigned c, unsigned cnt) {
    P.ctrl->segcnt[np][bin][c] = cnt;
    if constexpr (MG) s_wl_acc += cnt;
}

// Plain variant: push of a loser with cooperative conversion (one atomic per
// warp, IrGL's warp-aggregated push) into the bin's dense next list, in
// whatever order the warps arrive.  Called by the whole warp.
template <class F>
__device__ __forceinline__ void plain_push(const Params &P, int np, int bin, bool take, int u,
                                           unsigned long long od) {
    const unsigned m = __ballot_sync(FULL, take);
    if (!m) return;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane_id() == (unsigned)leader) base = atomicAdd(&P.ctrl->plain_cnt[np][bin], (unsigned long long)__popc(m));
    base = __shfl_sync(FULL, base, leader);
    if (take) {
        const unsigned long long pos = base + __popc(m & lanemask_lt());
        dyn_list(P, np, bin)[pos] = u;
        if constexpr (!F::small) dyn_od(P, np, bin)[pos] = od;
    }
}

// set by any thread of the CTA that issued NVLink stores in the current
// phase: only such CTAs need the system-scope fence before the next barrier
__shared__ unsigned s_mirrored;
// multi-GPU, per round: the boundary zones are copied to the peers at the end
// of each phase instead of mirroring every store (dense boundaries)
__shared__ unsigned s_bulk;

// Cross-GPU barrier of the multi-GPU solve: the grid barrier whose last
// arriving CTA exchanges (epoch, payload) with every rank's mailbox over
// NVLink.  kind 0: plain;  kind 1: end of round t with parity p -- payload =
// this rank's (|W_{t+1}|, conflicts of t), global sums left in C->g_wl /
// C->g_conf for the next round's mode decision (driver.py:147-152) and record.
// Every CTA fences its mirrored stores (fence.sc.sys) before arriving, so a
// peer that passes the barrier sees them.  Returns false if some rank did not
// arrive within P.timeout_ns (the whole grid then leaves the kernel).
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

template <class SMT>
__device__ bool mg_sync(const Params &P, SMT &sm, unsigned long long epoch, int kind, int p) {
    Ctrl *C = P.ctrl;
    GridBarrier *b = &C->bar;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_u32(&b->gen);
        if (s_mirrored) {  // this CTA's NVLink stores are ordered before its arrival
            fence_acq_rel_sys();
            s_mirrored = 0u;
        } else {
            __threadfence();
        }
        const unsigned arrived = atomicAdd(&b->count, 1u);
        if (arrived == P.nblocks - 1) {
            atomicExch(&b->count, 0u);
            unsigned long long a = 0, c = 0;
            if (kind == 1) {
                a = __ldcg(&C->wl_next[p ^ 1]) + __ldcg(&C->hub_cnt[p ^ 1]);
                c = __ldcg(&C->conflicts[p]);
            }
            unsigned long long sa = 0, sc = 0;
            unsigned ok = 1;
#if HC_MG_PLAIN_BARRIER  // experiment knob (valid for one rank only): no mailbox, no system fences
            sa = a;
            sc = c;
#else
            // release: everything this GPU wrote (observed through the
            // arrivals) before the tags; then relaxed tagged stores
            fence_acq_rel_sys();
            const unsigned long long tag = (epoch & 0xffffffffull) << 32;
            const unsigned long long wv[3] = {tag | (a & 0xffffffffull), tag | (c & 0xffffffffull), tag | (c >> 32)};
            const int par = (int)(epoch & 1ull);
            for (int q = 0; q < P.world; ++q) {
                MboxSlot *sl = &P.peer_mbox[q]->slot[par][P.rank];
#pragma unroll
                for (int w = 0; w < 3; ++w) st_relaxed_sys_u64(&sl->w[w], wv[w]);
            }
            const unsigned long long t0 = globaltimer();
            for (int q = 0; q < P.world && ok; ++q) {
                MboxSlot *sl = &P.mbox->slot[par][q];
#pragma unroll 1
                for (int w = 0; w < 3 && ok; ++w) {
                    unsigned long long v;
                    while (((v = ld_relaxed_sys_u64(&sl->w[w])) & ~0xffffffffull) != tag) {
                        if ((long long)(globaltimer() - t0) > P.timeout_ns) {
                            ok = 0;
                            break;
                        }
                        __nanosleep(20);
                    }
                    const unsigned long long val = v & 0xffffffffull;
                    if (w == 0) sa += val;
                    else if (w == 1) sc += val;
                    else sc += val << 32;
                }
            }
            fence_acq_rel_sys();  // acquire: the peers' data before the tags they posted
#endif
            if (!ok) C->abort = 1u;
            if (kind == 1) {
                C->g_wl = sa;
                C->g_conf = sc;
            }
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (ld_acquire_u32(&b->gen) == g) __nanosleep(20);
        }
        __threadfence();
        sm.mg_abort = *(volatile unsigned *)&C->abort;
    }
    __syncthreads();
    return sm.mg_abort == 0u;
}

// Storage formats, chosen per graph by hc_solve:
//   state word  XT = uint32 (bit 31 = committed)  or uint16 (bit 15), the
//               latter when max degree <= 16384 so every color fits 15 bits
//   column id   CT = int32 absolute  or int16 delta (v - u), the latter when
//               every |v - u| < 2^15 (grids / meshes with local numbering)
// All solver logic works on the 32-bit encoding; the accessors convert.
//   MG          multi-GPU (hc_mg_solve): this rank owns [lo, lo+nown); writes
//               of owned boundary words are mirrored into every peer's replica
//   SMALL       only bin-0 nodes (see SmemT)
//   PLAIN       bench-only "Plain" data-driven baseline (the paper's IrGL Plain,
//               PAPER.md:268-283): losers are pushed with warp-aggregated
//               atomics into one dense, unordered list per bin instead of the
//               order-preserving segmented compaction (_kernels.pyx:114-118)
//   ELL         bin-0-only graphs with every degree <= 4 and 16-bit deltas
//               (grids): a node's whole adjacency is one 8-byte word (Params
//               ell) loaded together with its state word -- no row offsets,
//               no dependent column load
//   LIVE        live lower lists (Params lc): resolve scans of bins 1..4 keep
//               only the still-uncolored lower neighbours (skewed graphs)
template <typename XT, typename CT, bool MG = false, bool SMALL = false, bool PLAIN = false, bool ELL = false,
          bool LIVEL = false>
struct Fmt {
    using xt = XT;
    using ct = CT;
    static constexpr bool mg = MG;
    static constexpr bool small = SMALL;
    static constexpr bool plain = PLAIN;
    static constexpr bool ell = ELL;
    static constexpr bool live = LIVEL;
    static_assert(!ELL || (SMALL && !MG && sizeof(CT) == 2), "ELL4 rows: bin-0-only, single GPU, delta columns");
    static_assert(!LIVEL || (!SMALL && !MG && !PLAIN), "live lower lists: general single-GPU kernel");
};
using F32 = Fmt<unsigned, int>;
using F16 = Fmt<unsigned short, int>;
using F16D = Fmt<unsigned short, short>;
using F32D = Fmt<unsigned, short>;
using MF32 = Fmt<unsigned, int, true>;
using MF16 = Fmt<unsigned short, int, true>;
using MF16D = Fmt<unsigned short, short, true>;
using MF32D = Fmt<unsigned, short, true>;
using SF32 = Fmt<unsigned, int, false, true>;
using SF16 = Fmt<unsigned short, int, false, true>;
using SF16D = Fmt<unsigned short, short, false, true>;
using SF32D = Fmt<unsigned, short, false, true>;
using SMF32 = Fmt<unsigned, int, true, true>;
using SMF16 = Fmt<unsigned short, int, true, true>;
using SMF16D = Fmt<unsigned short, short, true, true>;
using SMF32D = Fmt<unsigned, short, true, true>;
using PF32 = Fmt<unsigned, int, false, false, true>;
using PF16 = Fmt<unsigned short, int, false, false, true>;
using PF16D = Fmt<unsigned short, short, false, false, true>;
using PF32D = Fmt<unsigned, short, false, false, true>;
using PSF32 = Fmt<unsigned, int, false, true, true>;
using PSF16 = Fmt<unsigned short, int, false, true, true>;
using PSF16D = Fmt<unsigned short, short, false, true, true>;
using PSF32D = Fmt<unsigned, short, false, true, true>;
using SEF16D = Fmt<unsigned short, short, false, true, false, true>;
using SEF32D = Fmt<unsigned, short, false, true, false, true>;
using PSEF16D = Fmt<unsigned short, short, false, true, true, true>;
using PSEF32D = Fmt<unsigned, short, false, true, true, true>;
using LF32 = Fmt<unsigned, int, false, false, false, false, true>;
using LF16 = Fmt<unsigned short, int, false, false, false, false, true>;
using LF16D = Fmt<unsigned short, short, false, false, false, false, true>;
using LF32D = Fmt<unsigned, short, false, false, false, false, true>;
// 8-bit state words (colors <= 127): general-kernel graphs of max degree
// <= 128 (ER-2^25): the whole state array stays L2-resident at twice the node
// count.  (Bin-0-only graphs keep 16 bits: grid4096 measured 352 -> 355 ms.)
using F8 = Fmt<unsigned char, int>;
using F8D = Fmt<unsigned char, short>;
using PF8 = Fmt<unsigned char, int, false, false, true>;
using PF8D = Fmt<unsigned char, short, false, false, true>;

// committed flag / color mask of the format's state word; words are kept
// zero-extended in registers, so no conversion on load or store
template <class F>
constexpr unsigned FB = sizeof(typename F::xt) == 4 ? 0x80000000u : sizeof(typename F::xt) == 2 ? 0x8000u : 0x80u;
template <class F>
constexpr unsigned CM = FB<F> - 1u;

template <class F>
__device__ __forceinline__ unsigned xget(const Params &P, long long v) {
    return reinterpret_cast<const typename F::xt *>(P.X)[v];
}
// store to the local word only (initialisation)
template <class F>
__device__ __forceinline__ void xraw(const Params &P, long long v, unsigned w) {
    reinterpret_cast<typename F::xt *>(P.X)[v] = (typename F::xt)w;
}
// multi-GPU: the word of an owned boundary node is also stored into every
// peer's replica (NVLink stores; made visible by the fence.sys of the next
// cross-GPU barrier).  Interior words are read by no other rank.
// Only the ranks that read the word get it (bit q of the node's peer mask),
// and the mask is loaded only inside the boundary zones at the two ends of
// the owned range (an arithmetic test; grids: a few rows per cut).
template <class F>
__device__ __forceinline__ void mirror(const Params &P, long long v, unsigned w, unsigned mask) {
    s_mirrored = 1u;
    while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1u;
        reinterpret_cast<typename F::xt *>(__ldg(reinterpret_cast<const unsigned long long *>(P.peer_x) + q))[v] =
            (typename F::xt)w;
    }
}
template <class F>
__device__ __forceinline__ void xput(const Params &P, long long v, unsigned w) {
    reinterpret_cast<typename F::xt *>(P.X)[v] = (typename F::xt)w;
    if constexpr (F::mg) {
        if (!s_bulk && (v - P.lo < P.zlo || P.lo + P.nown - v <= P.zhi)) {
            const unsigned mask = __ldg(P.bnd + v);
            if (mask) mirror<F>(P, v, w, mask);
        }
    }
}
// Zone copy (bulk exchange): the prefix [lo, lo+zlo) goes to every lower rank
// and the suffix [hi-zhi, hi) to every higher rank -- every word a peer can
// read lies there (mg_boundary_kernel).  All CTAs, 16-byte vector stores.
template <class F>
__device__ void zone_copy(const Params &P) {
    using xt = typename F::xt;
    constexpr long long V = 16 / sizeof(xt);  // words per vector
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)P.nblocks * blockDim.x;
    const xt *src = reinterpret_cast<const xt *>(P.X);
    bool any = false;
    for (int q = 0; q < P.world; ++q) {
        if (q == P.rank) continue;
        const long long b = q < P.rank ? P.lo : P.lo + P.nown - P.zhi;
        const long long e = q < P.rank ? P.lo + P.zlo : P.lo + P.nown;
        if (e <= b) continue;
        any = true;
        xt *dst = reinterpret_cast<xt *>(__ldg(reinterpret_cast<const unsigned long long *>(P.peer_x) + q));
        const long long vb = (b + V - 1) / V, ve = e / V;  // whole vectors inside [b, e)
        if (vb < ve) {
            for (long long i = b + gtid; i < vb * V; i += gthreads) dst[i] = src[i];
            for (long long i = ve * V + gtid; i < e; i += gthreads) dst[i] = src[i];
            const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
            uint4 *d4 = reinterpret_cast<uint4 *>(dst);
            for (long long i = vb + gtid; i < ve; i += gthreads) d4[i] = __ldcg(s4 + i);
        } else {
            for (long long i = b + gtid; i < e; i += gthreads) dst[i] = src[i];
        }
    }
    if (any) s_mirrored = 1u;
}

// tentative color write: a 16-bit word cannot hold T > 32767 (possible only
// for degree > 32766); flag it, the host reruns the solve with 32-bit words
template <class F>
__device__ __forceinline__ void xput_t(const Params &P, long long v, unsigned T) {
    if (sizeof(typename F::xt) < 4 && T > CM<F>) *P.fmt_overflow = 1u;
    xput<F>(P, v, T);
}
// load of a column id.  Low-degree rows are streamed (evict-first, so the
// X gathers keep L2); hub / bin-3 rows (KEEP) are cached at L2 normally:
// the same hub adjacency is re-scanned in every round of the hub core.
template <class F, bool KEEP = false>
__device__ __forceinline__ int colget(const Params &P, long long k, int u) {
    if constexpr (sizeof(typename F::ct) == 4)
        return KEEP ? __ldcg(P.ci + k) : __ldcs(P.ci + k);
    else
        return u + (int)(KEEP ? __ldcg(P.ci16 + k) : __ldcs(P.ci16 + k));
}

// ELL4 word helpers: the word travels in TileA's (rb, re) register pair
template <typename OffT>
__device__ __forceinline__ unsigned long long ell_word(OffT lo, OffT hi) {
    return (unsigned long long)(unsigned)lo | ((unsigned long long)(unsigned)hi << 32);
}
__device__ __forceinline__ int ell_nb(unsigned long long w, int q, int u) {
    const short d = (short)(unsigned short)(w >> (16 * q));
    return d != 0 ? u + (int)d : -1;
}
__device__ __forceinline__ unsigned ell_deg(unsigned long long w) {
    unsigned d = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) d += ((w >> (16 * q)) & 0xffffull) != 0;
    return d;
}

template <class F>
__device__ __forceinline__ void mask_add(unsigned long long &mask, unsigned x) {
    const unsigned c = x & CM<F>;
    if ((x & FB<F>) && c <= 64u) mask |= 1ull << (c - 1u);
}

// ---------------------------------------------------- forbidden-color bitmaps
// A node's bitmap covers colors 1..deg+1 (its mex is <= deg+1,
// _kernels.pyx:49-56): word fb0[u] for colors 1..32, then floor(deg/32) words
// fbx[(ro[u] >> 5) ...] for colors 33.. -- disjoint per node because
// (ro[u+1] >> 5) - (ro[u] >> 5) >= floor(deg(u) / 32), so no per-node offset
// array is needed.  Bits are only ever set (by winners, in resolve), and assign
// of round t reads them after the grid barrier that ends round t-1: the bitmap
// then holds exactly the colors committed before round t, i.e. the
// reference's colors_read snapshot restricted to u's neighbours.
#ifndef HC_FBM
#define HC_FBM 1
#endif
template <class F>
constexpr bool FBM = HC_FBM && !F::mg;  // the multi-GPU solve keeps the adjacency-scan assign
template <class F>
constexpr bool LIVE = HC_LIVE && F::live;  // live lower lists (Params lc)

#ifndef HC_FB_FILTER
#define HC_FB_FILTER 1   // skip pushes into neighbours already committed (one X gather per push)
#endif
#ifndef HC_FB_HINT
#define HC_FB_HINT 1     // bitmap REDs with an L2 evict-first policy (keep the X gathers' lines)
#endif
__device__ __forceinline__ void fb_or(unsigned *a, unsigned bits) {
#if HC_FB_HINT
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "red.relaxed.gpu.global.or.L2::cache_hint.b32 [%0], %1, pol;\n\t}" ::"l"(a),
        "r"(bits)
        : "memory");
#else
    atomicOr(a, bits);
#endif
}

// winner's color c into neighbour v's bitmap (fire-and-forget RED).
// CHECK: v's word was not read yet -- with HC_FB_FILTER a committed v (whose
// bitmap is never read again) gets no push.  Not in the bin-0-only kernel:
// there a winner has at most a few unread (higher) neighbours and the
// dependent gather costs more than the extra REDs (grid4096 353.7 -> 350.1
// ms without it; ER-2^25 needs it: 46.6 vs 55.2 ms)
template <class F, bool CHECK = true, typename OffT>
__device__ __forceinline__ void fb_push(const Params &P, const OffT *ro, int v, unsigned c) {
    if constexpr (CHECK && HC_FB_FILTER && !F::small) {
        if (xget<F>(P, v) & FB<F>) return;
    }
    if (c <= 32u) {
        fb_or(P.fb0 + v, 1u << (c - 1u));
        return;
    }
    const long long b = (long long)ro[v], e = (long long)ro[v + 1];
    if ((long long)c > e - b + 1) return;  // c > deg(v)+1 is never v's mex
    fb_or(P.fbx + (b >> 5) + ((c - 33u) >> 5), 1u << ((c - 33u) & 31u));
}

// mex of node u's bitmap, one thread (w0 = fb0[u] already loaded)
template <typename OffT>
__device__ __forceinline__ unsigned fb_mex_thread(const Params &P, const OffT *ro, int u, unsigned w0) {
    if (w0 != FULL) return (unsigned)__ffs(~w0);
    const unsigned *x = P.fbx + ((long long)ro[u] >> 5);
    for (unsigned j = 0;; ++j) {  // a zero bit exists among colors 1..deg+1
        const unsigned w = x[j];
        if (w != FULL) return 32u * j + 32u + (unsigned)__ffs(~w);
    }
}

// mex of a hub / CTA-granularity node's bitmap, whole CTA
template <typename OffT, class SMT>
__device__ unsigned fb_mex_cta(const Params &P, const OffT *ro, int u, SMT &sm) {
    const unsigned w0 = P.fb0[u];
    if (w0 != FULL) return (unsigned)__ffs(~w0);
    const unsigned *x = P.fbx + ((long long)ro[u] >> 5);
    const long long nw = ((long long)ro[u + 1] >> 5) - ((long long)ro[u] >> 5);
    for (long long j0 = 0;; j0 += BLOCK) {
        if (threadIdx.x == 0) sm.hub_first = 0x7fffffff;
        __syncthreads();
        const long long j = j0 + threadIdx.x;
        if (j < nw && x[j] != FULL) atomicMin(&sm.hub_first, (int)(j - j0));
        __syncthreads();
        const int f = sm.hub_first;
        __syncthreads();
        if (f != 0x7fffffff) return 32u * (unsigned)(j0 + f) + 32u + (unsigned)__ffs(~x[j0 + f]);
    }
}

// a winner of the CTA-granularity paths pushes its color into every neighbour
// (PU column loads per thread in flight, then their state words, then the
// REDs: a hub's whole row is one pass of deg / (PU * BLOCK) round trips)
constexpr int PU = 8;
template <typename OffT, class F>
__device__ __forceinline__ void fb_push_row_cta(const Params &P, const OffT *ro, int u, unsigned c) {
#if HC_PHASE_TIMES
    const unsigned long long tp0 = globaltimer();
    struct TP {  // development builds: longest CTA push of the round (stats column 6)
        const Params &P;
        unsigned long long t0;
        __device__ ~TP() {
            if (threadIdx.x == 0 && P.stats && P.ctrl->rounds_live >= 1 && P.ctrl->rounds_live <= P.max_rec)
                atomicMax((unsigned long long *)&P.stats[5 * P.max_rec + 8 * (P.ctrl->rounds_live - 1) + 6],
                          globaltimer() - t0);
        }
    } tp{P, tp0};
#endif
    const long long b = ro[u], e = ro[u + 1];
    for (long long k0 = b + threadIdx.x; k0 < e; k0 += (long long)PU * BLOCK) {
        int v[PU];
        unsigned x[PU];
#pragma unroll
        for (int q = 0; q < PU; ++q) {
            const long long k = k0 + (long long)q * BLOCK;
            v[q] = k < e ? colget<F, true>(P, k, u) : -1;
        }
#pragma unroll
        for (int q = 0; q < PU; ++q) x[q] = v[q] >= 0 ? xget<F>(P, v[q]) : FB<F>;
#pragma unroll
        for (int q = 0; q < PU; ++q)
            if (!(x[q] & FB<F>)) fb_push<F, false>(P, ro, v[q], c);  // committed neighbours need none
    }
}

// A winning hub's pushes: queued for the whole grid at the start of the next
// round (one CTA walking a 10^4..10^6-entry row was the longest unit of the
// RMAT tail rounds), or pushed here when the queue is full.  CTA-uniform.
template <typename OffT, class F, class SMT>
__device__ __forceinline__ void hub_push(const Params &P, const OffT *ro, SMT &sm, int p, int u, unsigned c) {
    if constexpr (HC_DEFER_PUSH) {
        if ((long long)(ro[u + 1] - ro[u]) < (long long)HC_DEFER_MIN) {  // CTA-uniform
            fb_push_row_cta<OffT, F>(P, ro, u, c);
            return;
        }
        if (threadIdx.x == 0) {
            const unsigned i = atomicAdd(&P.ctrl->pend_cnt[p], 1u);
            if (i < (unsigned)MAX_PEND) P.ctrl->pend[p][i] = u;
            sm.hub_first = i < (unsigned)MAX_PEND ? 1 : 0;
        }
        __syncthreads();
        const bool queued = sm.hub_first == 1;
        __syncthreads();
        if (queued) return;
    }
    fb_push_row_cta<OffT, F>(P, ro, u, c);
}

// The queued hub pushes of the previous round (parity q), every CTA a
// contiguous share of the concatenated rows; the caller separates them from
// the next assign with a grid barrier.  The hub's color is its committed word.
template <typename OffT, class F, class SMT>
__device__ void run_pending_pushes(const Params &P, const OffT *ro, SMT &sm, int q, unsigned npend) {
    unsigned *pre = sm.hub_pre;  // scratch: the rows' prefix (hub split rebuilds it afterwards)
    for (unsigned i = threadIdx.x; i < npend; i += BLOCK) {
        const int h = __ldcg(&P.ctrl->pend[q][i]);
        pre[i + 1] = (unsigned)(ro[h + 1] - ro[h]);
    }
    if (threadIdx.x == 0) pre[0] = 0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (unsigned i = 1; i <= npend; ++i) pre[i] += pre[i - 1];
    __syncthreads();
    const unsigned long long total = pre[npend];
    const unsigned long long share = (total + P.nblocks - 1) / P.nblocks;
    const unsigned long long lo = min(total, (unsigned long long)blockIdx.x * share), hi = min(total, lo + share);
    unsigned hub = 0;
    for (unsigned long long g = lo + threadIdx.x; g < hi; g += BLOCK) {
        while (pre[hub + 1] <= g) ++hub;  // positions grow along the loop
        const int h = __ldcg(&P.ctrl->pend[q][hub]);
        const unsigned c = xget<F>(P, h) & CM<F>;
        fb_push<F>(P, ro, colget<F, true>(P, (long long)ro[h] + (long long)(g - pre[hub]), h), c);
    }
}

// ------------------------------------------------------------------ groups
// Warp-level mex over window(s) above color 64, for a node whose colors
// 1..64 are all taken (rare): whole warp, one node.
template <class F>
__device__ unsigned warp_mex_above64(const Params &P, int u, long long b, long long e, unsigned *bm,
                                     unsigned start) {
    const unsigned lane = lane_id();
    const unsigned lim = (unsigned)(e - b) + 1u;
    for (unsigned w0 = start;; w0 += WIN_WORDS * 32) {
        bm[lane] = 0u;
        __syncwarp();
        const unsigned hi = min(lim, w0 + WIN_WORDS * 32);
        for (long long k = b + lane; k < e; k += 32) {
            const unsigned x = xget<F>(P, colget<F>(P, k, u));
            const unsigned c = x & CM<F>;
            if ((x & FB<F>) && c > w0 && c <= hi) mark(bm, c - w0);
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

// Live-list compaction of one 4-slot batch of a group (LIVE resolve): the
// lower entries whose word is still uncolored go to lc[b + kept ...] (any
// order), group-wise prefix from ballots; `kept` is the group's running count.
// `idx0`: this lane's slot-0 index in the scanned list; when the source is
// lc itself an entry that does not move is not rewritten.
template <int G, class F>
__device__ __forceinline__ void live_keep(const Params &P, long long b, const int *nb, const unsigned *x, int u,
                                          unsigned gmask, unsigned &kept, bool in_place, unsigned idx0) {
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const bool keep = nb[q] < u && !(x[q] & FB<F>);
        const unsigned bal = __ballot_sync(FULL, keep) & gmask;
        const unsigned at = kept + __popc(bal & lt);
        if (keep && !(in_place && at == idx0 + q * G)) P.lc[b + at] = nb[q];
        kept += __popc(bal);
    }
}

// The list entry of a group tile's node: id, (offset, degree) and the
// node's own state word (activity / tentative color).  Fetched one tile ahead
// in resolve (group_sub) so the next tile's list round trip and own-word
// round trip overlap this tile's column and neighbour-word gathers; X[u] is
// written by u's own processing only, so the early read sees the same value.
struct GEntry {
    int u;
    unsigned xu;
    unsigned long long od;
};
template <int G, class F, int PHASE>
__device__ __forceinline__ GEntry group_fetch(const Params &P, const List &L, const unsigned *prefix,
                                              unsigned long long v0, unsigned long long hi, bool topo,
                                              unsigned &seg_hint) {
    const unsigned gi = lane_id() / G;
    const unsigned long long v = v0 + gi;
    // the list entry carries the adjacency range (no dependent row-offset load)
    // segment walk from the warp's hint (positions only grow along a chunk):
    // no per-node binary search over up to MAXSEG segment starts
    unsigned sg = seg_hint;
    const long long idx = v < hi ? list_index_walk(L, prefix, v, sg) : -1;
    seg_hint = __shfl_sync(FULL, sg, 0);  // lane 0 holds the tile's first (smallest) position
    GEntry g;
    g.u = idx >= 0 ? ld_entry(L.base + idx) : -1;
    g.od = idx >= 0 ? ld_od(L.od + idx) : 0ull;
    g.xu = ((topo || PHASE == 1) && g.u >= 0) ? xget<F>(P, g.u) : 0u;
    return g;
}

// One warp tile of a group bin: 32/G nodes, G lanes per node (`pre`: the
// tile's entries, already fetched by group_fetch; nullptr: fetch here).
template <int G, typename OffT, class F, bool STATS, int PHASE>
__device__ __forceinline__ void group_tile(const Params &P, const OffT *ro, const List &L,
                                           const unsigned *prefix, unsigned long long v0,
                                           unsigned long long hi, bool topo, int *out,
                                           unsigned long long *out_od, unsigned *out_cnt, unsigned *bm,
                                           unsigned &seg_hint,
                                           unsigned long long &my_conf, unsigned long long *my_edges,
                                           int np_plain = 0, int bin_plain = 0, const GEntry *pre = nullptr) {
    const unsigned lane = lane_id();
    const unsigned sub = lane % G, gi = lane / G;
    const GEntry g = pre ? *pre : group_fetch<G, F, PHASE>(P, L, prefix, v0, hi, topo, seg_hint);
    int u = g.u;
    const unsigned long long od = g.od;
    const unsigned xu = g.xu;
    if (topo && (xu & FB<F>)) u = -1;  // inactive (_kernels.pyx:76-77, 135-136)
    const long long b = u >= 0 ? od_off(od) : 0;
    const long long e = u >= 0 ? b + (long long)(od & 0xffffull) : 0;
    if constexpr (PHASE == 0 && FBM<F>) {
        // mex of the node's forbidden-color bitmap: word fb0[u] (one
        // transaction per group), the extension words only if colors 1..32
        // are all taken -- G words per step, first non-full word of the group
        const unsigned w0 = u >= 0 ? P.fb0[u] : 0u;
        bool need = u >= 0 && w0 == FULL;
        unsigned T = (u >= 0 && !need) ? (unsigned)__ffs(~w0) : 0u;
        const unsigned *fx = P.fbx + (b >> 5);
        for (unsigned j0 = 0; __any_sync(FULL, need); j0 += G) {
            const unsigned w = need ? fx[j0 + sub] : FULL;
            const unsigned bal = __ballot_sync(FULL, need && w != FULL);
            const unsigned gb = G == 32 ? bal : (bal >> (gi * G)) & ((1u << (G & 31)) - 1u);
            const int f = gb ? __ffs(gb) - 1 : 0;
            const unsigned wf = __shfl_sync(FULL, w, (G == 32 ? 0 : (int)(gi * G)) + f);
            if (need && gb) {
                T = 32u * (j0 + (unsigned)f) + 32u + (unsigned)__ffs(~wf);
                need = false;
            }
        }
        if (sub == 0 && u >= 0) {
            xput<F>(P, u, T);
            if (STATS) my_edges[0] += e - b;
        }
        return;
    }
    // live lower list (data-driven resolve): scan lc[b, b + live) -- all
    // below u, no exit test -- once u has been scanned (od carries the
    // count), else the row with the early exit; the still-uncolored entries
    // are compacted to lc[b, ...) and the loser's next od carries their count.
    // (Topology sweeps read the static od: the row, no compaction.)
    constexpr bool LV = LIVE<F> && PHASE == 1;
    const bool lcomp = LV && !topo && (G == 32 || HC_LIVE_GROUPS);
    const bool lsrc = lcomp && (od & OD_LIVE);
    const long long se = lsrc ? b + (long long)((od >> 48) & 0x7fffull) : e;  // end of the scanned range
    unsigned iters = (unsigned)((se - b + 4 * G - 1) / (4 * G));
    iters = __reduce_max_sync(FULL, iters);
    unsigned long long mask = 0, mask2 = 0;  // colors 1..64, 65..128 (mask2: G == 32 only)
    unsigned cnt = 0, low = 0;
    unsigned kept = 0;  // live entries written back (LV)
    const unsigned gmask_lv = (G == 32) ? FULL : (((1u << (G & 31)) - 1u) << (gi * G));
    bool stop = u < 0;
    // software pipeline: the column ids of iteration it+1 are in flight while
    // the X gathers of iteration it are issued
    const int pad = PHASE == 0 ? -1 : 0x7fffffff;
    int nb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long k = b + sub + q * G;
        nb[q] = (!stop && k < se) ? (lsrc ? __ldcg(P.lc + k) : colget<F>(P, k, u)) : pad;
    }
    if constexpr (G < 32) {
        // bins 1 and 2: degree <= 4G, so the first column batch is the whole
        // adjacency -- one straight pass, no next-batch registers
        unsigned x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = (PHASE == 0 ? nb[q] >= 0 : nb[q] < u) ? xget<F>(P, nb[q]) : 0u;
        if (PHASE == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) mask_add<F>(mask, x[q]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (nb[q] < u) { cnt += (x[q] & CM<F>) == xu; ++low; }
            if (LV && lcomp) live_keep<G, F>(P, b, nb, x, u, gmask_lv, kept, lsrc, sub);
        }
        iters = 0;  // the loop below is skipped
    }
    for (unsigned it = 0; it < iters; ++it) {
        int nx[4];
        const long long kn = b + (long long)(it + 1) * 4 * G + sub;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long k = kn + q * G;
            nx[q] = (!stop && k < se) ? (lsrc ? __ldcg(P.lc + k) : colget<F>(P, k, u)) : pad;
        }
        if (PHASE == 0) {
            unsigned x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = nb[q] >= 0 ? xget<F>(P, nb[q]) : 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q) mask_add<F>(mask, x[q]);
            if constexpr (G == 32) {  // warp per node: colors 65..128 too (hub-core nodes)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned c = x[q] & CM<F>;
                    if ((x[q] & FB<F>) && c > 64u && c <= 128u) mask2 |= 1ull << (c - 65u);
                }
            }
        } else {
            unsigned x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = nb[q] < u ? xget<F>(P, nb[q]) : 0u;
            bool ge = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (nb[q] < u) { cnt += (x[q] & CM<F>) == xu; ++low; }
                else if (nb[q] != 0x7fffffff) ge = true;
            }
            // in place: this batch's writes land below its own positions, the
            // next batch is already in registers (nx)
            if (LV && lcomp) live_keep<G, F>(P, b, nb, x, u, gmask_lv, kept, lsrc, it * 4u * G + sub);
            // adjacency sorted ascending (graph.py:193-197): once any lane of the
            // group saw a neighbour >= u, the group's later iterations are all >= u
            const unsigned bal = __ballot_sync(FULL, ge);
            const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (gi * G));
            if (bal & gmask) stop = true;
            if (__all_sync(FULL, stop)) break;
            if (stop) {
#pragma unroll
                for (int q = 0; q < 4; ++q) nx[q] = pad;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) nb[q] = nx[q];
    }
    if (PHASE == 0) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) mask |= __shfl_xor_sync(FULL, mask, o);
        if constexpr (G == 32) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mask2 |= __shfl_xor_sync(FULL, mask2, o);
        }
        unsigned T;
        if (mask != ~0ull) {
            T = (unsigned)__ffsll((long long)~mask);
        } else if (G == 32 && mask2 != ~0ull) {
            T = 64u + (unsigned)__ffsll((long long)~mask2);  // no second pass over the adjacency
        } else if (G < 32) {
            T = 65u;  // deg <= 64 and colors 1..64 all taken: exactly 64 neighbours
        } else {
            T = 0u;   // warp-uniform (one node per warp): fall back to bitmap windows
        }
        if (G == 32 && T == 0u && u >= 0) T = warp_mex_above64<F>(P, u, b, e, bm, 128u);
        if (sub == 0 && u >= 0) {
            xput<F>(P, u, T);
            if (STATS) my_edges[0] += e - b;
        }
    } else {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            cnt += __shfl_xor_sync(FULL, cnt, o);
            low += __shfl_xor_sync(FULL, low, o);
        }
        if (sub == 0 && u >= 0) {
            my_conf += cnt;
            if (STATS) my_edges[1] += low;
            if (cnt) {
                if constexpr (!F::plain) {
                    const unsigned pos = atomicAdd(out_cnt, 1u);  // the segment's global loser count
                    out[pos] = u;
                    out_od[pos] = (LV && lcomp) ? od_live(od, kept) : od;
                    // multi-GPU: a global segment count (group_sub) bypasses seg_put's tally
                    if (F::mg && !__isShared(out_cnt)) atomicAdd(&s_wl_acc, 1ull);
                }
            } else {
                xput<F>(P, u, xu | FB<F>);
            }
        }
        if constexpr (F::plain) plain_push<F>(P, np_plain, bin_plain, sub == 0 && u >= 0 && cnt != 0, u, od);
        if constexpr (FBM<F>) {
            if (u >= 0 && cnt == 0) {  // group-uniform: the winner's color goes into every neighbour's bitmap
                if constexpr (G < 32) {
                    // the committed-neighbour filter's word loads are issued
                    // together, before any RED (a RED between them would order
                    // the next load behind it: four dependent round trips)
                    int w[4];
                    if (lsrc) {  // nb held the live lower list: the whole row comes from the columns
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const long long k = b + sub + q * G;
                            w[q] = k < e ? colget<F>(P, k, u) : -1;
                        }
                    } else {  // the first column batch is the whole adjacency
#pragma unroll
                        for (int q = 0; q < 4; ++q) w[q] = nb[q] != 0x7fffffff ? nb[q] : -1;
                    }
                    unsigned xw[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) xw[q] = (HC_FB_FILTER && w[q] >= 0) ? xget<F>(P, w[q]) : 0u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (w[q] >= 0 && !(xw[q] & FB<F>)) fb_push<F, false>(P, ro, w[q], xu);
                } else {  // whole warp, one node: PU column loads per lane in flight
                    for (long long k0 = b + sub; k0 < e; k0 += (long long)PU * G) {
                        int w[PU];
                        unsigned xw[PU];
#pragma unroll
                        for (int q = 0; q < PU; ++q) {
                            const long long k = k0 + (long long)q * G;
                            w[q] = k < e ? colget<F>(P, k, u) : -1;
                        }
#pragma unroll
                        for (int q = 0; q < PU; ++q) xw[q] = w[q] >= 0 ? xget<F>(P, w[q]) : FB<F>;
#pragma unroll
                        for (int q = 0; q < PU; ++q)
                            if (!(xw[q] & FB<F>)) fb_push<F, false>(P, ro, w[q], xu);
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ hub (CTA)
template <typename OffT, class F>
__device__ unsigned assign_cta(const Params &P, const OffT *ro, int u, Smem &sm) {
    const long long b = ro[u], e = ro[u + 1];
    const unsigned lim = (unsigned)(e - b) + 1u;
    for (unsigned w0 = 0;; w0 += HUB_WORDS * 32) {
        for (int i = threadIdx.x; i < HUB_WORDS; i += BLOCK) sm.hub_bm[i] = 0u;
        if (threadIdx.x == 0) sm.hub_first = 0x7fffffff;
        __syncthreads();
        const unsigned hi = min(lim, w0 + HUB_WORDS * 32);
        // software pipeline: the column ids of the next iteration are in
        // flight while this iteration's neighbour words are gathered
        int v[HU];
#pragma unroll
        for (int q = 0; q < HU; ++q) {
            const long long k = b + threadIdx.x + q * BLOCK;
            v[q] = k < e ? colget<F, true>(P, k, u) : -1;
        }
        // colors w0+1 .. w0+64 (the common ones) go to a register mask,
        // OR-reduced per warp: one shared atomic per warp instead of one per
        // neighbour on the same few hot words
        unsigned long long low = 0, low2 = 0;
        for (long long k = b + threadIdx.x; k < e; k += HU * BLOCK) {
            int nv[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                const long long kn = k + (HU + q) * BLOCK;
                nv[q] = kn < e ? colget<F, true>(P, kn, u) : -1;
            }
            unsigned x[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) x[q] = v[q] >= 0 ? xget<F>(P, v[q]) : 0u;
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                const unsigned c = x[q] & CM<F>;
                if (!(x[q] & FB<F>) || c <= w0 || c > hi) continue;
                if (c <= w0 + 64u) low |= 1ull << (c - w0 - 1u);
                else if (c <= w0 + 128u) low2 |= 1ull << (c - w0 - 65u);
                else mark(sm.hub_bm, c - w0);
            }
#pragma unroll
            for (int q = 0; q < HU; ++q) v[q] = nv[q];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            low |= __shfl_xor_sync(FULL, low, o);
            low2 |= __shfl_xor_sync(FULL, low2, o);
        }
        if (lane_id() == 0) {
            if (low) {
                atomicOr(&sm.hub_bm[0], (unsigned)low);
                atomicOr(&sm.hub_bm[1], (unsigned)(low >> 32));
            }
            if (low2) {
                atomicOr(&sm.hub_bm[2], (unsigned)low2);
                atomicOr(&sm.hub_bm[3], (unsigned)(low2 >> 32));
            }
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

// lcu: u's live lower count (>= 0: scan lc[b, b + lcu), all below u), or -1
// (scan the row with the early exit).  compact: write the still-uncolored
// entries back to lc[b, ...) in place -- one CTA barrier per chunk set so no
// warp writes ahead of the entries another warp still has to read -- and
// return their count in kept_out (LIVE).
template <typename OffT, class F>
__device__ unsigned resolve_cta(const Params &P, const OffT *ro, int u, unsigned T, Smem &sm,
                                unsigned &lower_out, int lcu = -1, bool compact = false,
                                unsigned *kept_out = nullptr) {
    const long long b = ro[u], e = ro[u + 1];
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    const bool lsrc = LIVE<F> && lcu >= 0;  // CTA-uniform
    const long long se = lsrc ? b + lcu : e;
    if (threadIdx.x == 0) {
        sm.red = 0;
        sm.kcnt = 0;
    }
    __syncthreads();
    unsigned cnt = 0, low = 0;
    // software pipeline: the next chunk's column ids are in flight while
    // this chunk's words are gathered (the adjacency is sorted, so the scan
    // stops at the first chunk holding an id >= u)
    int v[HU];
#pragma unroll
    for (int q = 0; q < HU; ++q) {
        const long long k = b + (long long)warp * (32 * HU) + 32 * q + lane;
        v[q] = k < se ? (lsrc ? __ldcg(P.lc + k) : colget<F, true>(P, k, u)) : 0x7fffffff;
    }
    if (LIVE<F> && (lsrc || compact)) {  // CTA-uniform
        const long long nit = (se - b + 32LL * HU * NW - 1) / (32LL * HU * NW);
        const unsigned lt = lanemask_lt();
        // in place: every warp holds its first chunk before any warp writes
        // (later chunk sets are loaded before the barrier that ends the
        // previous iteration, and writes stay below the current set's end)
        if (lsrc) __syncthreads();
        for (long long it = 0; it < nit; ++it) {
            const long long k0 = b + it * 32LL * HU * NW + (long long)warp * (32 * HU);
            const bool more = lsrc || __all_sync(FULL, v[HU - 1] < u);  // this chunk is wholly below u
            int nv[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                const long long k = k0 + 32LL * HU * NW + 32 * q + lane;
                nv[q] = (more && k < se) ? (lsrc ? __ldcg(P.lc + k) : colget<F, true>(P, k, u)) : 0x7fffffff;
            }
            unsigned x[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) x[q] = v[q] < u ? xget<F>(P, v[q]) : 0u;
            bool stop = false;
            unsigned bal[HU], wk = 0;
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                if (v[q] < u) { cnt += (x[q] & CM<F>) == T; ++low; }
                else stop = true;
                bal[q] = __ballot_sync(FULL, compact && v[q] < u && !(x[q] & FB<F>));
                wk += __popc(bal[q]);
            }
            unsigned base = 0;
            if (lane == 0 && wk) base = atomicAdd(&sm.kcnt, wk);
            base = __shfl_sync(FULL, base, 0);
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                const unsigned at = base + __popc(bal[q] & lt);
                const long long src = k0 - b + 32 * q + lane;  // this entry's index
                if (((bal[q] >> lane) & 1u) && !(lsrc && (long long)at == src)) P.lc[b + at] = v[q];
                base += __popc(bal[q]);
            }
#pragma unroll
            for (int q = 0; q < HU; ++q) v[q] = nv[q];
            if (__syncthreads_or(stop)) break;  // later chunk sets are all >= u
        }
    } else {
        for (long long k0 = b + (long long)warp * (32 * HU); k0 < e; k0 += 32LL * HU * NW) {
            const bool more = __all_sync(FULL, v[HU - 1] < u);  // this chunk is wholly below u
            int nv[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                const long long k = k0 + 32LL * HU * NW + 32 * q + lane;
                nv[q] = (more && k < e) ? colget<F, true>(P, k, u) : 0x7fffffff;
            }
            unsigned x[HU];
#pragma unroll
            for (int q = 0; q < HU; ++q) x[q] = v[q] < u ? xget<F>(P, v[q]) : 0u;
            bool stop = false;
#pragma unroll
            for (int q = 0; q < HU; ++q) {
                if (v[q] < u) { cnt += (x[q] & CM<F>) == T; ++low; }
                else stop = true;
            }
#pragma unroll
            for (int q = 0; q < HU; ++q) v[q] = nv[q];
            if (__any_sync(FULL, stop)) break;  // later chunks are all >= u
        }
    }
    cnt = warp_sum(cnt);
    low = warp_sum(low);
    // counts packed: conflicts in the low 32 bits, lower-neighbour visits above
    if (lane == 0 && (cnt | low)) atomicAdd(&sm.red, (unsigned long long)cnt | ((unsigned long long)low << 32));
    __syncthreads();
    const unsigned long long r = sm.red;
    if (kept_out) *kept_out = sm.kcnt;
    __syncthreads();
    lower_out = (unsigned)(r >> 32);
    return (unsigned)r;
}

// ------------------------------------------------------------------ bin 0
// Thread per node, NP nodes per thread (NPT, or NPT_SMALL in the bin-0-only
// kernel).  A tile is issued (list entry, row offsets, activity / tentative
// word of its NP nodes: tile_issue) and then finished (first-four-neighbour
// column loads, X gathers, mex / conflict count, writes: tile_finish); all
// loads of one stage are issued before any is consumed.  (Issuing tile i+1
// before finishing tile i was measured slower: grid4096 609 -> 752+ ms.)
template <typename OffT, int NP>
struct TileA {
    int u[NP];
    OffT rb[NP], re[NP];
    unsigned xu[NP];
    unsigned w0[NP];  // forbidden-color word of the node (bitmap assign)
};

template <typename OffT, class F, int NP, int PHASE, bool STATS>
__device__ __forceinline__ void tile_issue(const Params &P, const OffT *ro, const RoundCfg &rc,
                                           const unsigned *prefix, unsigned long long base,
                                           unsigned long long hi, TileA<OffT, NP> &a, unsigned &seg) {
    // seg: segment-walk hint carried across the tiles of a chunk (positions grow)
    const List &L = rc.L[0];
    const bool topo = rc.topo, ident = rc.ident;
    if constexpr (PHASE == 0 && FBM<F> && !STATS) {
        // bitmap assign: list entry, then the activity word (topology sweep)
        // and the forbidden-color word together -- no row offsets, no columns
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
            a.u[j] = v < hi ? (ident ? (int)(P.lo + (long long)v) : ld_entry(L.base + list_index_walk(L, prefix, v, seg)))
                            : -1;
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            a.xu[j] = (topo && a.u[j] >= 0) ? xget<F>(P, a.u[j]) : 0u;
            a.w0[j] = a.u[j] >= 0 ? P.fb0[a.u[j]] : 0u;
        }
        return;
    }
    if constexpr (F::ell) {
        // ELL4 rows: the adjacency word is loaded together with the activity /
        // tentative word (one dependent round trip instead of offsets -> columns)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
            a.u[j] = v < hi ? (ident ? (int)(P.lo + (long long)v) : ld_entry(L.base + list_index_walk(L, prefix, v, seg)))
                            : -1;
        }
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const unsigned long long w = a.u[j] >= 0 ? __ldcs(P.ell + a.u[j]) : 0ull;
            a.rb[j] = (OffT)(unsigned)w;
            a.re[j] = (OffT)(unsigned)(w >> 32);
            a.xu[j] = ((topo || PHASE == 1) && a.u[j] >= 0) ? xget<F>(P, a.u[j]) : 0u;
            if constexpr (PHASE == 0 && FBM<F>) a.w0[j] = a.u[j] >= 0 ? P.fb0[a.u[j]] : 0u;
        }
        return;
    }
    // bin-0-only graphs (grids, meshes) read the row offsets: their lists are
    // nearly id-ordered, so the offsets are almost contiguous, and a 4-byte
    // list entry beats the 12-byte (id, od) pair (grid4096 data 843 vs 969 ms)
    if (ident || F::small) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
            a.u[j] = v < hi ? (ident ? (int)(P.lo + (long long)v) : ld_entry(L.base + list_index_walk(L, prefix, v, seg)))
                            : -1;
        }
        // the row offsets are loaded together with the activity word
        // (speculative for inactive nodes): one dependent round trip less
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            a.rb[j] = a.u[j] >= 0 ? ro[a.u[j]] : OffT(0);
            a.re[j] = a.u[j] >= 0 ? ro[a.u[j] + 1] : OffT(0);
        }
    } else {  // list entries carry (row offset, degree)
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const unsigned long long v = base + (unsigned long long)j * BLOCK + threadIdx.x;
            const long long idx = v < hi ? list_index_walk(L, prefix, v, seg) : -1;
            a.u[j] = idx >= 0 ? ld_entry(L.base + idx) : -1;
            const unsigned long long od = idx >= 0 ? ld_od(L.od + idx) : 0ull;
            a.rb[j] = (OffT)od_off(od);
            a.re[j] = a.rb[j] + (OffT)(od & 0xffffull);
        }
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) a.xu[j] = ((topo || PHASE == 1) && a.u[j] >= 0) ? xget<F>(P, a.u[j]) : 0u;
    if constexpr (PHASE == 0 && FBM<F>) {  // STATS builds (row offsets loaded for the edge count)
#pragma unroll
        for (int j = 0; j < NP; ++j) a.w0[j] = a.u[j] >= 0 ? P.fb0[a.u[j]] : 0u;
    }
}

template <typename OffT, class F, bool STATS, int PHASE, int NP>
__device__ __forceinline__ void tile_finish(const Params &P, const OffT *ro, const RoundCfg &rc, TileA<OffT, NP> &a,
                                            bool *lost, unsigned long long &my_conf, unsigned long long *my_edges) {
    int *u = a.u;
    OffT *rb = a.rb, *re = a.re;
    const unsigned *xu = a.xu;
#pragma unroll
    for (int j = 0; j < NP; ++j) lost[j] = false;
    if constexpr (PHASE == 0 && FBM<F>) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            if (u[j] < 0 || (rc.topo && (xu[j] & FB<F>))) {  // inactive (_kernels.pyx:76-77)
                u[j] = -1;
                continue;
            }
            // deg <= 16: at most 16 bits of fb0 are set, a zero bit exists
            xput<F>(P, u[j], fb_mex_thread(P, ro, u[j], a.w0[j]));
            if (STATS) my_edges[0] += F::ell ? ell_deg(ell_word(rb[j], re[j])) : (unsigned long long)(re[j] - rb[j]);
        }
        return;
    }
    if (rc.topo) {
#pragma unroll
        for (int j = 0; j < NP; ++j)
            if (xu[j] & FB<F>) { u[j] = -1; re[j] = rb[j]; }  // inactive (_kernels.pyx:76-77, 135-136)
    }
    int nb[NP][4];
    if constexpr (F::ell) {  // deg <= 4: the word is the whole adjacency
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) nb[j][q] = u[j] >= 0 ? ell_nb(ell_word(rb[j], re[j]), q, u[j]) : -1;
    } else {
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) nb[j][q] = rb[j] + q < re[j] ? colget<F>(P, rb[j] + q, u[j]) : -1;
    }
    if (PHASE == 0) {
        unsigned x[NP][4];
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) x[j][q] = nb[j][q] >= 0 ? xget<F>(P, nb[j][q]) : 0u;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            if (u[j] < 0) continue;
            unsigned long long mask = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) mask_add<F>(mask, x[j][q]);
            for (OffT k = rb[j] + 4; !F::ell && k < re[j]; k += 4) {  // deg 5..16
                int v2[4];
                unsigned x2[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? colget<F>(P, k + q, u[j]) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) x2[q] = v2[q] >= 0 ? xget<F>(P, v2[q]) : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) mask_add<F>(mask, x2[q]);
            }
            xput<F>(P, u[j], (unsigned)__ffsll((long long)~mask));  // deg <= 16: a zero bit exists
            if (STATS) my_edges[0] += F::ell ? ell_deg(ell_word(rb[j], re[j])) : (unsigned long long)(re[j] - rb[j]);
        }
    } else {
        unsigned x[NP][4];
#pragma unroll
        for (int j = 0; j < NP; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) x[j][q] = (nb[j][q] >= 0 && nb[j][q] < u[j]) ? xget<F>(P, nb[j][q]) : 0u;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            if (u[j] < 0) continue;
            const unsigned T = xu[j];
            unsigned cnt = 0, low = 0;
            bool stop = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (nb[j][q] >= 0 && nb[j][q] < u[j]) { cnt += (x[j][q] & CM<F>) == T; ++low; }
                else stop = true;
            }
            for (OffT k = rb[j] + 4; !F::ell && !stop && k < re[j]; k += 4) {
                int v2[4];
                unsigned x2[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? colget<F>(P, k + q, u[j]) : 0x7fffffff;
#pragma unroll
                for (int q = 0; q < 4; ++q) x2[q] = v2[q] < u[j] ? xget<F>(P, v2[q]) : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (v2[q] < u[j]) { cnt += (x2[q] & CM<F>) == T; ++low; }
                    else stop = true;  // adjacency sorted ascending (graph.py:193-197)
                }
            }
            my_conf += cnt;
            if (STATS) my_edges[1] += low;
            lost[j] = cnt != 0;
            if (!lost[j]) xput<F>(P, u[j], T | FB<F>);
        }
        if constexpr (FBM<F>) {
            // winners put their color into every neighbour's bitmap (once per
            // node per solve); a lower neighbour already seen committed needs none
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                if (u[j] < 0 || lost[j]) continue;
                const unsigned T = xu[j];
                if constexpr (F::small) {  // (no filter loads: the original order measured faster on the grid)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (nb[j][q] >= 0 && !(nb[j][q] < u[j] && (x[j][q] & FB<F>))) {
                            if (nb[j][q] < u[j]) fb_push<F, false>(P, ro, nb[j][q], T);  // word already read
                            else fb_push<F>(P, ro, nb[j][q], T);
                        }
                    for (OffT k = rb[j] + 4; !F::ell && k < re[j]; k += 4) {  // deg 5..16
                        int v2[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? colget<F>(P, k + q, u[j]) : -1;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (v2[q] >= 0) fb_push<F>(P, ro, v2[q], T);
                    }
                } else {
                    // the filter's word loads before any RED: a RED between
                    // them would order each load behind the last RED
                    unsigned xw[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)  // a lower neighbour's word was already read
                        xw[q] = nb[j][q] < 0 ? FB<F> : nb[j][q] < u[j] ? x[j][q] : HC_FB_FILTER ? xget<F>(P, nb[j][q]) : 0u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (!(xw[q] & FB<F>)) fb_push<F, false>(P, ro, nb[j][q], T);
                    for (OffT k = rb[j] + 4; k < re[j]; k += 4) {  // deg 5..16
                        int v2[4];
                        unsigned x2[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) v2[q] = k + q < re[j] ? colget<F>(P, k + q, u[j]) : -1;
#pragma unroll
                        for (int q = 0; q < 4; ++q) x2[q] = v2[q] < 0 ? FB<F> : HC_FB_FILTER ? xget<F>(P, v2[q]) : 0u;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (!(x2[q] & FB<F>)) fb_push<F, false>(P, ro, v2[q], T);
                    }
                }
            }
        }
    }
}

// a chunk of a group bin: warps take warp tiles of 32/G nodes round-robin
// A unit of a group bin: rc.su[bin] consecutive list positions (whole warp
// tiles of 32/G nodes, G lanes per node), warps take tiles round-robin.
// Units are smaller than the output segments (rc.csz, at most MAXSEG per
// bin), so the heaviest nodes of a round do not queue behind each other in
// one long chunk (RMAT-22: the longest bin-3 chunk took 100-345 us of a
// 120-410 us resolve phase); a loser goes to the segment of its position
// through the segment's global count (zeroed at the start of the round).
template <int G, typename OffT, class F, bool STATS, int PHASE>
__device__ __forceinline__ void group_sub(const Params &P, const OffT *ro, Smem &sm, int bin,
                                          unsigned i, int np, unsigned long long &my_conf,
                                          unsigned long long *my_edges) {
    const RoundCfg &rc = sm.rc;
    const unsigned warp = threadIdx.x >> 5;
    const unsigned csz = rc.csz[bin];
    // bin 3: the first k3 positions went to CTA-per-node units
    const unsigned long long off = bin == 3 ? rc.k3 : 0u;
    const unsigned long long lo = off + (unsigned long long)i * rc.su[bin];
    const unsigned long long hi = min(lo + rc.su[bin], rc.L[bin].total);
    constexpr unsigned NG = 32 / G;
    // unit == segment (bins 1, 2): the CTA counts its losers in shared
    // memory and writes the segment's count once (bin 3: global counts; its
    // warp tiles are single nodes, so none straddles a segment)
    const bool whole = bin != 3 && rc.su[bin] == csz;
    if (whole) {
        if (threadIdx.x == 0) sm.out_cnt = 0;
        __syncthreads();
    }
    unsigned seg = lo < hi ? list_segment(rc.L[bin], sm.prefix[bin], lo) : 0u;  // once per unit
    constexpr unsigned long long STEP = (unsigned long long)NW * NG;
    if constexpr (PHASE == 1 && HC_GROUP_PREFETCH) {
        // resolve: the next tile's entries are fetched before this tile runs
        unsigned long long v0 = lo + (unsigned long long)warp * NG;
        GEntry cur{-1, 0u, 0ull};
        if (v0 < hi) cur = group_fetch<G, F, PHASE>(P, rc.L[bin], sm.prefix[bin], v0, hi, rc.topo, seg);
        for (; v0 < hi; v0 += STEP) {  // warp-uniform
            GEntry nxt{-1, 0u, 0ull};
            if (v0 + STEP < hi) nxt = group_fetch<G, F, PHASE>(P, rc.L[bin], sm.prefix[bin], v0 + STEP, hi, rc.topo, seg);
            const unsigned c = (unsigned)v0 / csz;  // a warp tile never straddles segments (csz: whole tiles); 32-bit: positions < 2^31
            group_tile<G, OffT, F, STATS, PHASE>(P, ro, rc.L[bin], sm.prefix[bin], v0, hi, rc.topo,
                                              dyn_list(P, np, bin) + (long long)c * csz,
                                              dyn_od(P, np, bin) + (long long)c * csz,
                                              whole ? &sm.out_cnt : &P.ctrl->segcnt[np][bin][c],
                                              sm.win_bm[warp], seg, my_conf, my_edges, np, bin, &cur);
            cur = nxt;
        }
    } else {
        for (unsigned long long v0 = lo + (unsigned long long)warp * NG; v0 < hi; v0 += STEP) {
            const unsigned c = (unsigned)v0 / csz;  // a warp tile never straddles segments (csz: whole tiles); 32-bit: positions < 2^31
            group_tile<G, OffT, F, STATS, PHASE>(P, ro, rc.L[bin], sm.prefix[bin], v0, hi, rc.topo,
                                              dyn_list(P, np, bin) + (long long)c * csz,
                                              dyn_od(P, np, bin) + (long long)c * csz,
                                              whole ? &sm.out_cnt : &P.ctrl->segcnt[np][bin][c],
                                              sm.win_bm[warp], seg, my_conf, my_edges, np, bin);
        }
    }
    if (whole) {
        __syncthreads();
        if (!F::plain && PHASE == 1 && threadIdx.x == 0) seg_put<F::mg>(P, np, bin, i, sm.out_cnt);
    }
}

// ------------------------------------------------------------------ split hubs
// Slice `slice` of k of hub u's adjacency, one CTA.  Partial results merge
// into the hub's global slot; the last slice to arrive finalizes (mex /
// winner-loser decision) and resets the slot for the next round.
template <typename OffT, class F>
__device__ unsigned assign_slice(const Params &P, const OffT *ro, int u, unsigned slice, unsigned k,
                                 HubAcc &acc, Smem &sm, bool &last) {
    const long long b0 = ro[u], e0 = ro[u + 1], len = e0 - b0;
    const long long b = b0 + len * slice / k, e = b0 + len * (slice + 1) / k;
    for (int i = threadIdx.x; i < HA_WORDS + 2; i += BLOCK) sm.hub_bm[i] = 0u;  // [0,1]: mask, [2..]: words
    __syncthreads();
    unsigned long long mask = 0;
    int v[HU];  // software pipeline as in assign_cta
#pragma unroll
    for (int q = 0; q < HU; ++q) {
        const long long kk = b + threadIdx.x + q * BLOCK;
        v[q] = kk < e ? colget<F, true>(P, kk, u) : -1;
    }
    for (long long kk = b + threadIdx.x; kk < e; kk += HU * BLOCK) {
        int nv[HU];
#pragma unroll
        for (int q = 0; q < HU; ++q) {
            const long long kn = kk + (HU + q) * BLOCK;
            nv[q] = kn < e ? colget<F, true>(P, kn, u) : -1;
        }
        unsigned x[HU];
#pragma unroll
        for (int q = 0; q < HU; ++q) x[q] = v[q] >= 0 ? xget<F>(P, v[q]) : 0u;
#pragma unroll
        for (int q = 0; q < HU; ++q) {
            const unsigned c = x[q] & CM<F>;
            if (!(x[q] & FB<F>)) continue;
            if (c <= 64u) mask |= 1ull << (c - 1u);
            else if (c <= 64u + 32u * HA_WORDS) mark(sm.hub_bm + 2, c - 64u);
        }
#pragma unroll
        for (int q = 0; q < HU; ++q) v[q] = nv[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mask |= __shfl_xor_sync(FULL, mask, o);
    if (lane_id() == 0 && mask) {
        atomicOr(&sm.hub_bm[0], (unsigned)mask);
        atomicOr(&sm.hub_bm[1], (unsigned)(mask >> 32));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long m = (unsigned long long)sm.hub_bm[0] | ((unsigned long long)sm.hub_bm[1] << 32);
        if (m) atomicOr(&acc.mask, m);
    }
    for (int i = threadIdx.x; i < HA_WORDS; i += BLOCK)
        if (sm.hub_bm[2 + i]) atomicOr(&acc.words[i], sm.hub_bm[2 + i]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        sm.hub_first = atomicAdd(&acc.arrive, 1u) == k - 1 ? 1 : 0;
    }
    __syncthreads();
    last = sm.hub_first == 1;
    __syncthreads();  // every thread has read the flag before thread 0 reuses it
    unsigned T = 0;
    if (last) {  // CTA-uniform
        __threadfence();
        if (threadIdx.x == 0) {
            const unsigned long long m = __ldcg(&acc.mask);
            if (m != ~0ull) {
                T = (unsigned)__ffsll((long long)~m);
            } else {
                for (int i = 0; i < HA_WORDS && !T; ++i) {
                    const unsigned w = __ldcg(&acc.words[i]);
                    if (w != FULL) T = 64u + 32u * i + (unsigned)__ffs(~w);
                }
            }
            sm.hub_first = (int)T;  // 0: every color <= 2048 taken
            acc.mask = 0;
            for (int i = 0; i < HA_WORDS; ++i) acc.words[i] = 0;
            acc.arrive = 0;
        }
        __syncthreads();
        T = (unsigned)sm.hub_first;
        __syncthreads();
        if (T == 0) T = assign_cta<OffT, F>(P, ro, u, sm);  // exact full scan (colors > 2048)
    }
    return T;
}

template <typename OffT, class F>
__device__ unsigned resolve_slice(const Params &P, const OffT *ro, int u, unsigned T, unsigned slice, unsigned k,
                                  HubAcc &acc, Smem &sm, bool &last, unsigned &low_out) {
    // a hub already scanned once splits its live lower list lc[b0, b0 + lcnt)
    // (all below u; read-only here: slices of other CTAs cannot compact in place)
    const int lcu = LIVE<F> ? __ldcg(P.lcnt + u) : -1;
    const bool lsrc = lcu >= 0;
    const long long b0 = ro[u], e0 = lsrc ? b0 + lcu : ro[u + 1], len = e0 - b0;
    const long long b = b0 + len * slice / k, e = b0 + len * (slice + 1) / k;
    const unsigned warp = threadIdx.x >> 5, lane = lane_id();
    unsigned cnt = 0, low = 0;
    // software pipeline: the next chunk's column ids are in flight while
    // this chunk's words are gathered (the adjacency is sorted, so the scan
    // stops at the first chunk holding an id >= u)
    int v[HU];
#pragma unroll
    for (int q = 0; q < HU; ++q) {
        const long long kk = b + (long long)warp * (32 * HU) + 32 * q + lane;
        v[q] = kk < e ? (lsrc ? __ldcg(P.lc + kk) : colget<F, true>(P, kk, u)) : 0x7fffffff;
    }
    for (long long k0 = b + (long long)warp * (32 * HU); k0 < e; k0 += 32LL * HU * NW) {
        const bool more = __all_sync(FULL, v[HU - 1] < u);  // this chunk is wholly below u
        int nv[HU];
#pragma unroll
        for (int q = 0; q < HU; ++q) {
            const long long kk = k0 + 32LL * HU * NW + 32 * q + lane;
            nv[q] = (more && kk < e) ? (lsrc ? __ldcg(P.lc + kk) : colget<F, true>(P, kk, u)) : 0x7fffffff;
        }
        unsigned x[HU];
#pragma unroll
        for (int q = 0; q < HU; ++q) x[q] = v[q] < u ? xget<F>(P, v[q]) : 0u;
        bool stop = false;
#pragma unroll
        for (int q = 0; q < HU; ++q) {
            if (v[q] < u) { cnt += (x[q] & CM<F>) == T; ++low; }
            else stop = true;
        }
#pragma unroll
        for (int q = 0; q < HU; ++q) v[q] = nv[q];
        if (__any_sync(FULL, stop)) break;  // adjacency sorted: the rest is >= u
    }
    cnt = warp_sum(cnt);
    low = warp_sum(low);
    if (lane == 0 && (cnt | low)) {
        atomicAdd(&acc.cnt, cnt);
        atomicAdd(&acc.low, low);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        sm.hub_first = atomicAdd(&acc.arrive, 1u) == k - 1 ? 1 : 0;
    }
    __syncthreads();
    last = sm.hub_first == 1;
    __syncthreads();
    unsigned total = 0;
    if (last) {
        __threadfence();
        total = __ldcg(&acc.cnt);
        low_out = __ldcg(&acc.low);
        __syncthreads();
        if (threadIdx.x == 0) {
            acc.cnt = 0;
            acc.low = 0;
            acc.arrive = 0;
        }
    }
    return total;
}

template <typename OffT, class F, bool STATS, int PHASE>
__device__ __forceinline__ void small_tile(const Params &P, const OffT *ro, const RoundCfg &rc,
                                           const unsigned *prefix, unsigned long long base,
                                           unsigned long long hi, TileA<OffT, F::small ? NPT_SMALL : NPT> &a,
                                           bool *lost, unsigned long long &my_conf, unsigned long long *my_edges,
                                           unsigned &seg) {
    constexpr int NP = F::small ? NPT_SMALL : NPT;
    tile_issue<OffT, F, NP, PHASE, STATS>(P, ro, rc, prefix, base, hi, a, seg);
    tile_finish<OffT, F, STATS, PHASE, NP>(P, ro, rc, a, lost, my_conf, my_edges);
}

// A chunk of bin 0 (thread per node, NP nodes per thread per tile).
template <typename OffT, class F, bool STATS, int PHASE, class SMT>
__device__ __forceinline__ void bin0_chunk(const Params &P, const OffT *ro, SMT &sm, unsigned c, int np,
                                           unsigned long long &my_conf, unsigned long long *my_edges) {
    constexpr int NP = F::small ? NPT_SMALL : NPT;
    const RoundCfg &rc = sm.rc;
    const unsigned csz0 = rc.csz[0];
    const unsigned long long lo = (unsigned long long)c * csz0;
    const unsigned long long hi = min(lo + csz0, rc.L[0].total);
    int *out = dyn_list(P, np, 0) + (long long)c * csz0;
    unsigned long long *out_od = dyn_od(P, np, 0) + (long long)c * csz0;
    // order-preserving compaction of the losers (index order j-major, then
    // thread), ONE barrier per tile: every warp publishes its per-j loser
    // counts into a double-buffered table and scans it itself.  (Order only
    // affects locality, but an unordered list fragments round after round.)
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned written = 0, buf = 0;
    // one segment search per chunk, then walks (not one search per tile)
    unsigned seg = (rc.ident || lo >= hi) ? 0u : list_segment(rc.L[0], sm.prefix[0], lo);
    // the bin-0-only kernel compacts PAIR tiles per barrier
    constexpr int PAIR = F::small ? HC_PAIR : 1;
    constexpr int NS = PAIR * NP;  // slices per compaction
    static_assert(NS <= 2 * NPT_MAX && NS <= 32, "cnt_tab holds 2*NPT_MAX slices, one per lane");
    constexpr unsigned long long STEP = (unsigned long long)BLOCK * NP;
    for (unsigned long long base = lo; base < hi; base += STEP * PAIR) {
        int u[NS];
        bool lost[NS];
        unsigned long long odv[F::small ? 1 : NS];  // (offset, degree) of the losers (general kernel)
#pragma unroll
        for (int t = 0; t < PAIR; ++t) {
            TileA<OffT, NP> cur;
            bool lt[NP];
            if (t == 0 || base + t * STEP < hi) {  // CTA-uniform
                small_tile<OffT, F, STATS, PHASE>(P, ro, rc, sm.prefix[0], base + t * STEP, hi, cur, lt, my_conf,
                                                  my_edges, seg);
            } else {
#pragma unroll
                for (int q = 0; q < NP; ++q) { cur.u[q] = -1; lt[q] = false; }
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                u[t * NP + q] = cur.u[q];
                lost[t * NP + q] = lt[q];
                if constexpr (!F::small && PHASE == 1) odv[t * NP + q] = make_od(cur.rb[q], cur.re[q]);
            }
        }
        if constexpr (PHASE == 1 && F::plain) {
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                unsigned long long odj = 0;
                if constexpr (!F::small) odj = odv[j];
                plain_push<F>(P, np, 0, lost[j], u[j], odj);
            }
        } else if (PHASE == 1) {
            unsigned bal[NS];
#pragma unroll
            for (int j = 0; j < NS; ++j) bal[j] = __ballot_sync(FULL, lost[j]);
            if (lane < NS) {
                unsigned mine = 0;
#pragma unroll
                for (int j = 0; j < NS; ++j)
                    if (lane == (unsigned)j) mine = __popc(bal[j]);
                sm.cnt_tab[buf][lane * NW + warp] = mine;
            }
            __syncthreads();
            unsigned run = written;
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                const unsigned v = lane < NW ? sm.cnt_tab[buf][j * NW + lane] : 0u;
                const unsigned before = __reduce_add_sync(FULL, lane < warp ? v : 0u);  // warps < me in slice j
                const unsigned tot_j = __reduce_add_sync(FULL, v);
                if (lost[j]) {
                    const unsigned pos = run + before + __popc(bal[j] & lanemask_lt());
                    out[pos] = u[j];
                    if constexpr (!F::small) out_od[pos] = odv[j];
                }
                run += tot_j;
            }
            written = run;
            buf ^= 1u;
        }
    }
    if (!F::plain && PHASE == 1 && threadIdx.x == 0) seg_put<F::mg>(P, np, 0, c, written);
}

// One unit of one phase.  All CTA-uniform inputs come from shared memory.
// Unit ranges: [ubase0, ubase1) hubs, then bins 3, 2, 1, 0.
template <typename OffT, class F, bool STATS, int PHASE, class SMT>
__device__ __forceinline__ void run_unit(const Params &P, const OffT *ro, SMT &sm, unsigned unit,
                                         int p, unsigned long long &my_conf,
                                         unsigned long long *my_edges) {
    const RoundCfg &rc = sm.rc;
    const int np = p ^ 1;
    if constexpr (F::small) {  // only bin-0 units exist
        bin0_chunk<OffT, F, STATS, PHASE>(P, ro, sm, unit - rc.ubase[4], np, my_conf, my_edges);
        return;
    } else {
    const unsigned *ub = rc.ubase;
    const bool is_hub = unit < ub[1];
    if (is_hub && rc.hub_split) {
        // ---- hub split into equal-size edge slices (few active hubs)
        unsigned lo = 0, hi = rc.L[BIN_HUB].total;  // hub with hub_pre[i] <= unit < hub_pre[i+1]
        while (hi - lo > 1) {
            const unsigned mid = (lo + hi) >> 1;
            if (sm.hub_pre[mid] <= unit) lo = mid;
            else hi = mid;
        }
        const unsigned slot = lo, slice = unit - sm.hub_pre[lo], k = sm.hub_pre[lo + 1] - sm.hub_pre[lo];
        const int u = rc.L[BIN_HUB].base[slot];
        const unsigned xu = xget<F>(P, u);
        if (rc.topo && (xu & FB<F>)) return;  // topology sweep: inactive (_kernels.pyx:76)
        HubAcc &acc = P.hub_acc[slot];
        bool last;
        if (PHASE == 0 && FBM<F>) {  // bitmap mex: no edge work to split, slice 0 assigns
            if (slice == 0) {
                const unsigned T = fb_mex_cta(P, ro, u, sm);
                if (threadIdx.x == 0) {
                    xput_t<F>(P, u, T);
                    if (STATS) my_edges[0] += ro[u + 1] - ro[u];
                }
            }
        } else if (PHASE == 0) {
            const unsigned T = assign_slice<OffT, F>(P, ro, u, slice, k, acc, sm, last);
            if (last && threadIdx.x == 0) {
                xput_t<F>(P, u, T);
                if (STATS) my_edges[0] += ro[u + 1] - ro[u];
            }
        } else {
            unsigned low = 0;
            const unsigned kc = resolve_slice<OffT, F>(P, ro, u, xu, slice, k, acc, sm, last, low);
            if (last && threadIdx.x == 0) {
                my_conf += kc;
                if (STATS) my_edges[1] += low;
                if (kc) dyn_list(P, np, BIN_HUB)[atomicAdd(&P.ctrl->hub_cnt[np], 1ull)] = u;
                else xput<F>(P, u, xu | FB<F>);
            }
            if constexpr (FBM<F>) {
                if (last && kc == 0) hub_push<OffT, F>(P, ro, sm, p, u, xu);  // CTA-uniform
            }
        }
        return;
    }
    if (is_hub || unit < ub[1] + rc.k3) {
        // ---- hub, or one of the first k3 bin-3 nodes (the heaviest: the
        //      lists run in descending degree buckets), or every bin-3 node
        //      in the latency regime: one CTA per node
        const unsigned c = is_hub ? unit : unit - ub[1];
        const long long li = is_hub ? (long long)c : list_index(rc.L[3], sm.prefix[3], c);
        const int u = is_hub ? rc.L[BIN_HUB].base[c] : rc.L[3].base[li];
        const unsigned xu = xget<F>(P, u);
        unsigned pushed = 0;
        // live lower list: hubs keep the count in lcnt (any round); bin-3
        // nodes in the list entry's od (data rounds; compaction there only)
        int lcu = -1;
        bool comp = false;
        unsigned long long od3 = 0;
        if (LIVE<F> && PHASE == 1) {
            if (is_hub) {
                lcu = __ldcg(P.lcnt + u);
                comp = true;
            } else if (!rc.topo) {
                od3 = ld_od(rc.L[3].od + li);
                lcu = (od3 & OD_LIVE) ? (int)((od3 >> 48) & 0x7fffull) : -1;
                comp = true;
            }
        }
        if (!(rc.topo && (xu & FB<F>))) {  // topology sweep: inactive (_kernels.pyx:76)
            if (PHASE == 0) {
                unsigned T;
                if constexpr (FBM<F>) T = fb_mex_cta(P, ro, u, sm);
                else T = assign_cta<OffT, F>(P, ro, u, sm);
                if (threadIdx.x == 0) {
                    xput_t<F>(P, u, T);
                    if (STATS) my_edges[0] += ro[u + 1] - ro[u];
                }
            } else {
                unsigned low, kept = 0;
                const unsigned k = resolve_cta<OffT, F>(P, ro, u, xu, sm, low, lcu, comp, &kept);
                // a loser's next entry carries its live count (a winner's list is never read again)
                const unsigned long long od_next = comp ? od_live(make_od(ro[u], ro[u + 1]), kept)
                                                        : make_od(ro[u], ro[u + 1]);
                if (threadIdx.x == 0) {
                    my_conf += k;
                    if (STATS) my_edges[1] += low;
                    if (k) {
                        if (is_hub) {
                            if (comp) P.lcnt[u] = (int)kept;
                            dyn_list(P, np, BIN_HUB)[atomicAdd(&P.ctrl->hub_cnt[np], 1ull)] = u;
                        } else if constexpr (F::plain) {
                            const unsigned long long pos = atomicAdd(&P.ctrl->plain_cnt[np][3], 1ull);
                            dyn_list(P, np, 3)[pos] = u;
                            dyn_od(P, np, 3)[pos] = make_od(ro[u], ro[u + 1]);
                        } else if (rc.bin3_by_cta) {  // segment c, capacity 1
                            dyn_list(P, np, 3)[c] = u;
                            dyn_od(P, np, 3)[c] = od_next;
                        } else {  // the segment of position c, through its global count
                            const unsigned sgm = c / rc.csz[3];
                            const long long at = (long long)sgm * rc.csz[3] + atomicAdd(&P.ctrl->segcnt[np][3][sgm], 1u);
                            dyn_list(P, np, 3)[at] = u;
                            dyn_od(P, np, 3)[at] = od_next;
                            if constexpr (F::mg) s_wl_acc += 1ull;
                        }
                        pushed = 1;
                    } else {
                        xput<F>(P, u, xu | FB<F>);
                    }
                }
                if constexpr (FBM<F>) {
                    if (k == 0) {  // CTA-uniform
                        if (is_hub) hub_push<OffT, F>(P, ro, sm, p, u, xu);
                        else fb_push_row_cta<OffT, F>(P, ro, u, xu);
                    }
                }
            }
        }
        if (!F::plain && !is_hub && rc.bin3_by_cta && PHASE == 1 && threadIdx.x == 0) seg_put<F::mg>(P, np, 3, c, pushed);
    } else if (unit < ub[2]) {
        group_sub<32, OffT, F, STATS, PHASE>(P, ro, sm, 3, unit - ub[1] - rc.k3, np, my_conf, my_edges);
    } else if (unit < ub[3]) {
        group_sub<16, OffT, F, STATS, PHASE>(P, ro, sm, 2, unit - ub[2], np, my_conf, my_edges);
    } else if (unit < ub[4]) {
        group_sub<8, OffT, F, STATS, PHASE>(P, ro, sm, 1, unit - ub[3], np, my_conf, my_edges);
    } else {
        bin0_chunk<OffT, F, STATS, PHASE>(P, ro, sm, unit - ub[4], np, my_conf, my_edges);
    }
    }
}

// One bitmap-assign unit (phase 0 with forbidden-color bitmaps, rc.abase):
// a hub (the CTA takes the mex of its bitmap) or BLOCK * NPA consecutive
// entries of one bin's list, thread per node: list entry -> (activity word,
// bitmap word fb0) -> tentative word.  No row offsets, no columns (a node whose
// colors 1..32 are all taken reads its fbx words, fb_mex_thread).
template <typename OffT, class F, class SMT>
__device__ __forceinline__ void assign_unit(const Params &P, const OffT *ro, SMT &sm, unsigned unit) {
    const RoundCfg &rc = sm.rc;
    const unsigned *ab = rc.abase;
    const bool topo = rc.topo;
    if (unit < ab[1]) {  // hub (CTA-uniform)
        if constexpr (!F::small) {
            const int u = rc.L[BIN_HUB].base[unit];
            if (topo && (xget<F>(P, u) & FB<F>)) return;  // inactive (_kernels.pyx:76)
            const unsigned T = fb_mex_cta(P, ro, u, sm);
            if (threadIdx.x == 0) xput_t<F>(P, u, T);
        }
        return;
    }
    int b = 3;
    while (unit >= ab[5 - b]) --b;  // bins 3, 2, 1, 0 in unit order
    constexpr int NA = F::small ? HC_NPA_SMALL : HC_NPA;
    constexpr unsigned long long ACH = (unsigned long long)BLOCK * NA;
    const List &L = rc.L[b];
    const unsigned *prefix = sm.prefix[F::small ? 0 : b];
    const unsigned long long lo = (unsigned long long)(unit - ab[4 - b]) * ACH;
    const unsigned long long hi = min(lo + ACH, L.total);
    const bool ident = b == 0 && rc.ident;
    unsigned seg = (ident || lo >= hi) ? 0u : list_segment(L, prefix, lo);
    int u[NA];
    unsigned xu[NA], w0[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        const unsigned long long v = lo + (unsigned long long)j * BLOCK + threadIdx.x;
        u[j] = v < hi ? (ident ? (int)(P.lo + (long long)v) : ld_entry(L.base + list_index_walk(L, prefix, v, seg)))
                      : -1;
    }
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        xu[j] = (topo && u[j] >= 0) ? xget<F>(P, u[j]) : 0u;
        w0[j] = u[j] >= 0 ? P.fb0[u[j]] : 0u;
    }
#pragma unroll
    for (int j = 0; j < NA; ++j) {
        if (u[j] < 0 || (topo && (xu[j] & FB<F>))) continue;  // inactive (_kernels.pyx:76-77)
        xput_t<F>(P, u[j], fb_mex_thread(P, ro, u[j], w0[j]));
    }
}

template <typename OffT, class F, bool STATS, int PHASE, class SMT>
__device__ __forceinline__ void run_phase(const Params &P, const OffT *ro, SMT &sm, int p,
                                          unsigned long long &my_conf, unsigned long long *my_edges) {
    // bitmap assign: its own unit space (no output lists; STATS builds keep
    // the binned path, which also counts the assign edges)
    constexpr bool FA = PHASE == 0 && FBM<F> && (!STATS || HC_PHASE_TIMES);  // (timing builds: the production assign)
    unsigned *ctr = &P.ctrl->unit_ctr[PHASE][p];
    if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);
    __syncthreads();
    unsigned unit = sm.unit;
    const unsigned nunits = FA ? sm.rc.abase[NBIN] : sm.rc.ubase[NBIN];
    __syncthreads();
#if HC_PHASE_TIMES
    unsigned long long busy = 0;
    const long long t_round = STATS ? (long long)sm.rc.round : 0;
#endif
    while (unit < nunits) {
        if (threadIdx.x == 0) sm.unit = atomicAdd(ctr, 1u);  // prefetch the next unit
#if HC_PHASE_TIMES
        const unsigned long long t0 = globaltimer();
#endif
        if constexpr (FA) assign_unit<OffT, F>(P, ro, sm, unit);
        else run_unit<OffT, F, STATS, PHASE>(P, ro, sm, unit, p, my_conf, my_edges);
        __syncthreads();
#if HC_PHASE_TIMES
        // development builds, resolve: longest unit per kind (hub, bin 3..0)
        // and the busiest CTA, per round, behind the (start, assign, resolve) times
        if (STATS && PHASE == 1 && threadIdx.x == 0 && t_round >= 1 && t_round <= P.max_rec) {
            const unsigned long long d = globaltimer() - t0;
            busy += d;
            int kind = 0;
            while (kind < NBIN - 1 && unit >= sm.rc.ubase[kind + 1]) ++kind;
            atomicMax((unsigned long long *)&P.stats[5 * P.max_rec + 8 * (t_round - 1) + kind], d);
        }
#endif
        unit = sm.unit;
        __syncthreads();
    }
#if HC_PHASE_TIMES
    if (STATS && PHASE == 1 && threadIdx.x == 0 && t_round >= 1 && t_round <= P.max_rec)
        atomicMax((unsigned long long *)&P.stats[5 * P.max_rec + 8 * (t_round - 1) + 5], busy);
#endif
}

// ------------------------------------------------------------------ kernel
template <typename OffT, class F, bool STATS>
__global__ void __launch_bounds__(BLOCK, F::small ? MIN_CTAS_SMALL : MIN_CTAS) solve_kernel(Params P) {
    constexpr int NSB = F::small ? 1 : NSEG_BINS;  // segmented bins present
    __shared__ SmemT<F::small> sm;
    Ctrl *C = P.ctrl;
    const OffT *ro = reinterpret_cast<const OffT *>(P.ro);
    const unsigned lane = lane_id();
    const unsigned warp = threadIdx.x >> 5;
    const long long gtid = (long long)blockIdx.x * BLOCK + threadIdx.x;
    const long long gthreads = (long long)P.nblocks * BLOCK;
    RoundCfg &rc = sm.rc;

    for (long long u = gtid; u < P.n; u += gthreads) {
        xraw<F>(P, u, 0u);
        if constexpr (FBM<F>) P.fb0[u] = 0u;
    }
    if (threadIdx.x == 0) {
        unsigned long long off = 0;
        for (int b = 0; b < NBIN; ++b) {
            rc.nst[b] = C->nstat[b];
            rc.stat_lists[b] = P.stat + off;
            rc.stat_od[b] = P.stat_od + off;
            off += rc.nst[b];
        }
        rc.ident_small = rc.nst[0] == (unsigned long long)P.nown;  // all nodes in bin 0: sweep ids
        for (int b = 0; b < NSEG_BINS; ++b) rc.prev_nseg[b] = rc.prev_cap[b] = 0;
    }
    // multi-GPU: barrier epochs continue from the previous solve (every rank
    // runs the same number of barriers); the first barrier also guarantees
    // every replica is zeroed before any peer mirrors into it
    unsigned long long ep = 0;
    if constexpr (F::mg) {
        if (threadIdx.x == 0) {
            s_mirrored = 0u;
            s_wl_acc = 0ull;
            s_bulk = 0u;
        }
        ep = *(volatile unsigned long long *)&P.mbox->last_epoch;
        if (!mg_sync(P, sm, ++ep, 0, 0)) return;
    } else {
        grid_sync(&C->bar, P.nblocks);
    }

    unsigned long long t_start = 0;  // block 0 / thread 0 record keeping
    long long wl_in_prev = 0;
    int topo_prev = 0;
    unsigned long long my_conf = 0;
    unsigned long long my_edges[2] = {0, 0};  // stats: assign edges, resolve lower edges
    long long t = 1;
    for (;; ++t) {
        const int p = (int)(t & 1), np = p ^ 1;
        // ---- current worklist sizes: rebuild the segment prefix of the
        //      previous round's output (round 1: the full static lists)
        if (!F::plain && t > 1) {
            // bins with at most 32 segments (every bin in the latency regime):
            // one warp each scans them with shuffles -- no CTA barriers
            // (general kernel only: the bin-0-only kernel measured slower with it)
            if (!F::small && warp < (unsigned)NSB) {
                const unsigned ns = rc.prev_nseg[warp];
                if (ns <= 32u) {
                    const unsigned v = lane < ns ? __ldcg(&C->segcnt[p][warp][lane]) : 0u;
                    const unsigned vi = warp_incl_scan(v);
                    if (lane < ns) sm.prefix[warp][lane + 1] = vi;
                    if (lane == 0) sm.prefix[warp][0] = 0;
                }
            }
            bool big = F::small;
#pragma unroll
            for (int b = 0; b < NSB; ++b) big = big || rc.prev_nseg[b] > 32u;
            if (!big) __syncthreads();
#pragma unroll 1
            for (int b = 0; big && b < NSB; ++b) {
                const unsigned ns = rc.prev_nseg[b];
                if (!F::small && ns <= 32u) continue;  // CTA-uniform: scanned by its warp above (before this loop's barriers)
                for (unsigned s = threadIdx.x; s < ns; s += BLOCK)
                    sm.prefix[b][s + 1] = __ldcg(&C->segcnt[p][b][s]);
                if (threadIdx.x == 0) sm.prefix[b][0] = 0;
                __syncthreads();
                // inclusive scan of prefix[1..ns] (ns <= MAXSEG), PPT items per thread
                constexpr int PPT = MAXSEG / BLOCK;
                unsigned a[PPT], sum = 0;
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const unsigned i = 1 + PPT * threadIdx.x + q;
                    a[q] = i <= ns ? sm.prefix[b][i] : 0u;
                    sum += a[q];
                }
                const unsigned incl = warp_incl_scan(sum);
                if (lane == 31) sm.warp_tmp[warp] = incl;
                __syncthreads();
                if (warp == 0) {
                    const unsigned v = lane < NW ? sm.warp_tmp[lane] : 0u;
                    const unsigned vi = warp_incl_scan(v);
                    if (lane < NW) sm.warp_tmp[lane] = vi - v;
                }
                __syncthreads();
                unsigned run = sm.warp_tmp[warp] + incl - sum;
#pragma unroll
                for (int q = 0; q < PPT; ++q) {
                    const unsigned i = 1 + PPT * threadIdx.x + q;
                    run += a[q];
                    if (i <= ns) sm.prefix[b][i] = run;
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) {
            for (int b = 0; b < NSEG_BINS; ++b) {
                if (F::small && b > 0) {  // empty bins (SmemT<true> keeps one prefix)
                    rc.L[b] = List{rc.stat_lists[b], rc.stat_od[b], 0, 0, 0, false};
                    continue;
                }
                if constexpr (F::plain)  // dense, unordered lists of the previous round's pushes
                    rc.L[b] = t == 1 ? List{rc.stat_lists[b], rc.stat_od[b], rc.nst[b], 0, 0, false}
                                     : List{dyn_list(P, p, b), dyn_od(P, p, b), ld_relaxed_u64(&C->plain_cnt[p][b]), 0,
                                            0, false};
                else
                    rc.L[b] = t == 1 ? List{rc.stat_lists[b], rc.stat_od[b], rc.nst[b], 0, 0, false}
                                     : List{dyn_list(P, p, b), dyn_od(P, p, b), sm.prefix[F::small ? 0 : b][rc.prev_nseg[b]],
                                            rc.prev_nseg[b], rc.prev_cap[b], true};
            }
            const unsigned long long hub_total = t == 1 ? rc.nst[BIN_HUB] : ld_relaxed_u64(&C->hub_cnt[p]);
            rc.L[BIN_HUB] = List{t == 1 ? rc.stat_lists[BIN_HUB] : dyn_list(P, p, BIN_HUB), nullptr, hub_total, 0, 0,
                                 false};
            unsigned long long s = 0;  // this rank's |W_t| (the whole |W_t| on one GPU)
            for (int b = 0; b < NBIN; ++b) s += rc.L[b].total;
            // global |W_t|: multi-GPU sums over ranks at the end-of-round barrier
            const unsigned long long sg = !F::mg ? s : t == 1 ? (unsigned long long)P.n : __ldcg(&C->g_wl);
            const bool topo = P.mode == HC_MODE_TOPO || (P.mode == HC_MODE_HYBRID && (long long)sg > P.thr);
            // bin-3 nodes at CTA granularity when few are active (latency regime)
            const bool bin3_cta = HC_BIN3_CTA && rc.L[3].total <= 2ull * P.nblocks;
            if (topo)  // topology-driven: sweep the static lists, activity test
                for (int b = 0; b < NBIN; ++b)
                    rc.L[b] = List{rc.stat_lists[b], rc.stat_od[b], rc.nst[b], 0, 0, false};
            rc.topo = topo;
            rc.round = t;
            rc.ident = topo && rc.ident_small;
            if constexpr (F::mg) {
                // bulk when copying the zones (plus the extra local barrier it
                // needs, ~2 MB of link time) is cheaper than mirroring the
                // expected boundary stores of the round (~32 B per scattered
                // peer store; the active set is assumed boundary-proportional)
                const double zbytes =
                    ((double)P.zlo * P.rank + (double)P.zhi * (P.world - 1 - P.rank)) * sizeof(typename F::xt);
                const double mbytes = (double)s * (double)P.peer_words / (double)max(P.nown, 1LL) * 32.0;
                rc.bulk = P.world > 1 && (P.exchange == 2 || (P.exchange == 0 && zbytes + 2097152.0 < mbytes));
                s_bulk = rc.bulk ? 1u : 0u;
            }
            rc.csz[0] = chunk_size(rc.L[0].total, BLOCK * (F::small ? NPT_SMALL : NPT));
            rc.csz[1] = chunk_size(rc.L[1].total, NW * 4);
            rc.csz[2] = chunk_size(rc.L[2].total, NW * 2);
            rc.csz[3] = (bin3_cta && rc.L[3].total <= MAXSEG) ? 1u : chunk_size(rc.L[3].total, NW);
            // (32-bit divisions: list totals are < 2^31, and thread 0's
            // arithmetic here is on every round's critical path)
            for (int b = 0; b < NSEG_BINS; ++b)
                rc.nch[b] = ((unsigned)rc.L[b].total + rc.csz[b] - 1u) / rc.csz[b];
            rc.bin3_by_cta = rc.csz[3] == 1u;
            // group-bin work units: whole warp tiles, about UPC per CTA at most;
            // bin 3 (degrees 65..4096) keeps one tile per unit up to 64 per CTA
#pragma unroll
            for (int b = 1; b < NSEG_BINS; ++b) {
                // bins 1, 2 (similar degrees): unit = segment; bin 3 (65..4096):
                // about HC_UPC3 units per CTA, at least one warp tile each
                const unsigned tile = NW * (b == 1 ? 4u : b == 2 ? 2u : 1u);
                const unsigned tot = (unsigned)rc.L[b].total;
                const unsigned tiles = (tot + tile - 1u) / tile;
                unsigned k = b == 3 ? tiles / ((unsigned)HC_UPC3 * P.nblocks) : ~0u;
                k = max(1u, min(k, rc.csz[b] / tile));
                rc.su[b] = (b == 3 && rc.bin3_by_cta) ? 1u : k * tile;
                rc.nsu[b] = (tot + rc.su[b] - 1u) / rc.su[b];
            }
            // the heaviest bin-3 nodes (list front) one CTA each: a single
            // degree-4096 node would hold a warp ~28 us (RMAT-16 resolve)
            rc.k3 = rc.bin3_by_cta ? (unsigned)rc.L[3].total
                                   : (unsigned)min(rc.L[3].total, (unsigned long long)(P.nblocks * HC_K3 / 100));
            if (!rc.bin3_by_cta)
                rc.nsu[3] = ((unsigned)rc.L[3].total - rc.k3 + rc.su[3] - 1u) / rc.su[3];
            else
                rc.nsu[3] = 0;
            const bool live = s != 0;
            rc.ubase[0] = 0;
            // few active hubs (< nblocks): split them into edge slices; the
            // slice prefix is built below by the whole CTA
            const unsigned H = (unsigned)rc.L[BIN_HUB].total;
            rc.hub_split = (!HC_NO_SPLIT && live && H > 0 && (HC_SPLIT_ANY || H < P.nblocks) && H <= MAX_SPLIT_SLOTS) ? 1u : 0u;
            rc.ubase[1] = live ? H : 0u;
            rc.ubase[2] = rc.ubase[1] + (live ? rc.k3 + rc.nsu[3] : 0u);
            rc.ubase[3] = rc.ubase[2] + (live ? rc.nsu[2] : 0u);
            rc.ubase[4] = rc.ubase[3] + (live ? rc.nsu[1] : 0u);
            rc.ubase[5] = rc.ubase[4] + (live ? rc.nch[0] : 0u);
            {  // bitmap-assign units: one per hub, then BLOCK * NPA nodes per chunk of bins 3..0
                constexpr unsigned ACH = BLOCK * (F::small ? HC_NPA_SMALL : HC_NPA);
                rc.abase[0] = 0;
                rc.abase[1] = live ? H : 0u;
                for (int b = 3; b >= 0; --b)
                    rc.abase[5 - b] = rc.abase[4 - b] + (live ? (unsigned)((rc.L[b].total + ACH - 1) / ACH) : 0u);
            }
            // a tentative color overflowed the 16-bit state word: stop now (the
            // host redoes the solve with 32-bit words), never loop on a
            // truncated color
            sm.red = (!F::mg && __ldcg(P.fmt_overflow)) ? 0ull : sg;  // broadcast |W_t|
            // every round commits at least the lowest-id active node, so a
            // solve has at most n rounds; more means a broken invariant --
            // stop (HC_ERR_STALLED) instead of looping forever
            if (t > P.n + 1) {
                sm.red = 0ull;
                if (blockIdx.x == 0) C->rec_overflow = 2;
            }
            if (blockIdx.x == 0) {
                const unsigned long long now = globaltimer();
                if (t > 1) {  // finish the record of round t-1 (driver.py:159-168)
                    const int q = np;
                    if (t - 1 <= P.max_rec) {
                        hc_round_rec r;
                        r.round = t - 1;
                        r.topo = topo_prev;
                        r.wl_in = wl_in_prev;
                        r.wl_out = (long long)sg;
                        r.conflicts = F::mg ? (long long)__ldcg(&C->g_conf) : (long long)C->conflicts[q];
                        r.ns = (long long)(now - t_start);
                        P.rec[t - 2] = r;
                    }
                    C->conflicts[q] = 0;
                    C->hub_cnt[q] = 0;
                    if constexpr (F::plain)
                        for (int b = 0; b < NSEG_BINS; ++b) C->plain_cnt[q][b] = 0;
                    C->wl_next[q] = 0;
                    C->unit_ctr[0][q] = C->unit_ctr[1][q] = 0;
                }
                t_start = now;
#if HC_PHASE_TIMES
                C->rounds_live = t;
                if (STATS && t <= P.max_rec) P.stats[2 * P.max_rec + 3 * (t - 1)] = (long long)now;
#endif
                wl_in_prev = (long long)sg;
                topo_prev = topo;
            }
        }
        __syncthreads();
        const unsigned long long s = sm.red;
        __syncthreads();
        if (s == 0) break;  // worklist drained (driver.py:145)
        if (F::mg && blockIdx.x == 0 && threadIdx.x == 0) C->rounds = t;  // progress (timeout report)
        if constexpr (!F::small && !F::plain) {
            // the group bins' output segments collect their losers with global
            // counts (group_sub): zero this round's (parity np; their last
            // reader was the prefix rebuild of round t-1, the resolve that
            // fills them is behind the next grid barrier)
            for (int b = 1; b < NSEG_BINS; ++b)
                for (long long i = gtid; i < (long long)rc.nch[b]; i += gthreads) C->segcnt[np][b][i] = 0u;
        }
        if constexpr (FBM<F> && !F::small && HC_DEFER_PUSH) {
            // the previous round's winning hubs: their pushes, shared by every
            // CTA, then a barrier so this round's assign sees them
            const unsigned npend = t > 1 ? min(__ldcg(&C->pend_cnt[np]), (unsigned)MAX_PEND) : 0u;
            if (npend) {  // CTA-uniform
                run_pending_pushes<OffT, F>(P, ro, sm, np, npend);
                grid_sync(&C->bar, P.nblocks);
                if (blockIdx.x == 0 && threadIdx.x == 0) C->pend_cnt[np] = 0;
            }
        }
        if (!F::small && rc.hub_split) {  // CTA-uniform: equal-size edge slices over the active hubs
            const unsigned H = (unsigned)rc.L[BIN_HUB].total;
            unsigned long long e_loc = 0;
            for (unsigned i = threadIdx.x; i < H; i += BLOCK) {
                const int u = rc.L[BIN_HUB].base[i];
                const int lcu = (LIVE<F> && FBM<F>) ? __ldcg(P.lcnt + u) : -1;  // resolve slices split the live list
                e_loc += lcu >= 0 ? (unsigned long long)lcu : (unsigned long long)(ro[u + 1] - ro[u]);
            }
            e_loc = warp_sum(e_loc);
            if (threadIdx.x == 0) sm.red = 0;
            __syncthreads();
            if (lane == 0 && e_loc) atomicAdd(&sm.red, e_loc);
            __syncthreads();
            // ~2 slices per CTA in total, at least 4096 edges each
            const unsigned long long S = max(4096ull, (sm.red + 2ull * P.nblocks - 1) / (2ull * P.nblocks));
            for (unsigned i = threadIdx.x; i < H; i += BLOCK) {
                const int u = rc.L[BIN_HUB].base[i];
                const int lcu = (LIVE<F> && FBM<F>) ? __ldcg(P.lcnt + u) : -1;
                const unsigned long long d = lcu >= 0 ? (unsigned long long)lcu : (unsigned long long)(ro[u + 1] - ro[u]);
                sm.hub_pre[i + 1] = (unsigned)max(1ull, (d + S - 1) / S);
            }
            if (threadIdx.x == 0) sm.hub_pre[0] = 0;
            __syncthreads();
            if (warp == 0) {  // H < nblocks <= a few hundred: warp scan, 32 slots per step
                unsigned carry = 0;
                for (unsigned i0 = 1; i0 <= H; i0 += 32) {
                    const unsigned i = i0 + lane;
                    const unsigned v = i <= H ? sm.hub_pre[i] : 0u;
                    const unsigned incl = warp_incl_scan(v) + carry;
                    if (i <= H) sm.hub_pre[i] = incl;
                    carry = __shfl_sync(FULL, incl, 31);
                }
                if (lane == 0) {
                    const unsigned extra = carry - H;
                    for (int b = 1; b <= NBIN; ++b) rc.ubase[b] += extra;
                }
            }
            __syncthreads();
        }

        run_phase<OffT, F, STATS, 0>(P, ro, sm, p, my_conf, my_edges);
        if constexpr (F::mg) {
            if (rc.bulk) {  // every local word of the phase written, then the zones go out
                grid_sync(&C->bar, P.nblocks);
                zone_copy<F>(P);
            }
            if (!mg_sync(P, sm, ++ep, 0, p)) return;  // peers' tentative colors are in
        } else {
            grid_sync(&C->bar, P.nblocks);
        }
#if HC_PHASE_TIMES
        // development builds: per round (start, assign end, resolve end) in
        // globaltimer ns, behind the 2 * max_rec edge counters
        if (STATS && blockIdx.x == 0 && threadIdx.x == 0 && t <= P.max_rec)
            P.stats[2 * P.max_rec + 3 * (t - 1) + 1] = (long long)globaltimer();
#endif
        run_phase<OffT, F, STATS, 1>(P, ro, sm, p, my_conf, my_edges);

        // conflicts of this round: block reduce then one atomic per CTA
        {
            unsigned long long v = warp_sum(my_conf);
            my_conf = 0;
            if (threadIdx.x == 0) sm.red = 0;
            __syncthreads();
            if (lane == 0 && v) atomicAdd(&sm.red, v);
            __syncthreads();
            if (threadIdx.x == 0 && sm.red) atomicAdd(&C->conflicts[p], sm.red);
            if (F::mg && threadIdx.x == 0) {  // (only thread 0 touches the tally here)
                const unsigned long long w = s_wl_acc;
                if (w) {
                    atomicAdd(&C->wl_next[np], w);
                    s_wl_acc = 0ull;
                }
            }
            if (STATS) {
                for (int q = 0; q < 2; ++q) {
                    const unsigned long long e = warp_sum(my_edges[q]);
                    my_edges[q] = 0;
                    if (lane == 0 && e && t <= P.max_rec)
                        atomicAdd((unsigned long long *)&P.stats[2 * (t - 1) + q], e);
                }
            }
        }
        if (threadIdx.x == 0)
            for (int b = 0; b < NSEG_BINS; ++b) {
                rc.prev_nseg[b] = rc.nch[b];
                rc.prev_cap[b] = rc.csz[b];
            }
        if constexpr (F::mg) {
            if (rc.bulk) {
                grid_sync(&C->bar, P.nblocks);
                zone_copy<F>(P);
            }
            if (!mg_sync(P, sm, ++ep, 1, p)) return;  // winners in; global (|W'|, conflicts)
        } else {
            grid_sync(&C->bar, P.nblocks);
        }
#if HC_PHASE_TIMES
        if (STATS && blockIdx.x == 0 && threadIdx.x == 0 && t <= P.max_rec)
            P.stats[2 * P.max_rec + 3 * (t - 1) + 2] = (long long)globaltimer();
#endif
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->rounds = t - 1;
        if (t - 1 > P.max_rec && C->rec_overflow == 0) C->rec_overflow = 1;
        if constexpr (F::mg) P.mbox->last_epoch = ep;
    }
    for (long long i = gtid; i < P.nown; i += gthreads)
        P.colors_out[i] = (long long)(xget<F>(P, P.lo + i) & CM<F>);
}

// host stub address of one solve_kernel instantiation (explicitly
// instantiated per group in hcb_solve_inst.cu)
template <typename OffT, class F, bool STATS>
const void *kernel_ptr() {
    return (const void *)solve_kernel<OffT, F, STATS>;
}

// every instantiation, by group: X(offset type, format, stats)
#define HC_SIX(X, FAM, ST) \
    X(long long, FAM##F16, ST) X(long long, FAM##F32, ST) X(int, FAM##F16D, ST) X(int, FAM##F16, ST) \
    X(int, FAM##F32D, ST) X(int, FAM##F32, ST)
#define HC_INST_G0(X) HC_SIX(X, , false)
#define HC_INST_G1(X) HC_SIX(X, , true)
#define HC_INST_G2(X) HC_SIX(X, S, false)
#define HC_INST_G3(X) HC_SIX(X, S, true)
#define HC_INST_G4(X) HC_SIX(X, P, false)
#define HC_INST_G5(X) HC_SIX(X, PS, false)
#define HC_INST_G6(X) HC_SIX(X, M, false)
#define HC_INST_G7(X) HC_SIX(X, SM, false)
#define HC_INST_G8(X) \
    X(int, SEF16D, false) X(int, SEF32D, false) X(int, SEF16D, true) X(int, SEF32D, true) X(int, PSEF16D, false) \
    X(int, PSEF32D, false)
#define HC_INST_G9(X) HC_SIX(X, L, false)
#define HC_INST_G10(X) HC_SIX(X, L, true)
#define HC_INST_G11(X) X(int, F8, false) X(int, F8D, false) X(int, PF8, false) X(int, PF8D, false)
#define HC_INST_ALL(X) \
    HC_INST_G0(X) HC_INST_G1(X) HC_INST_G2(X) HC_INST_G3(X) HC_INST_G4(X) HC_INST_G5(X) HC_INST_G6(X) HC_INST_G7(X) \
    HC_INST_G8(X) HC_INST_G9(X) HC_INST_G10(X) HC_INST_G11(X)

}  // namespace solve
}  // namespace hcb
