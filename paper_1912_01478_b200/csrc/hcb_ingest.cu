// hcb_ingest.cu -- graph ingestion and degree statistics on the device
// (SURVEY.md §8(f) #2 / #3).
//
// MatrixMarket entries (reference graph.py:105-181, parse_matrix_market).
// The host parses the banner and the size line (a few bytes; exact reference
// messages) and hands the rest of the file, as raw bytes in HBM, to
// hc_mtx_parse:
//   1. line terminators: ordered compaction of the byte positions holding
//      '\n' (and '\r' for files read with universal newlines)
//   2. entry lines: ordered compaction of the lines whose first
//      non-whitespace byte exists and is not '%' (comments / blank lines are
//      skipped, graph.py:155-157)
//   3. one thread per entry line: first two whitespace-separated fields
//      (str.split semantics), Python int() syntax (sign, digits, single
//      underscores between digits), bounds 1..rows / 1..cols, ordinal < nnz;
//      entry k writes edges[k] = (r-1, c-1).
// Errors are ranked by line: the first offending line wins, exactly as the
// reference's sequential loop raises at the first bad line (graph.py:158-
// 176).  The device returns (line, code); the host formats the message from
// that one line.
//
// Degree statistics (graph.py:204-217, degree_stats): min, max and the
// element at sorted index n/2 (np.partition) by a 3-pass radix select over
// 11/11/9-bit digits of the degree, with shared-memory histograms.
#include <algorithm>

#include "hcb_partition.cuh"

namespace hcb {
namespace ingest {

__device__ __forceinline__ bool is_term(unsigned char c, bool cr) { return c == '\n' || (cr && c == '\r'); }
// ASCII whitespace of Python's str.split(): \t \n \v \f \r, \x1c-\x1f, space
__device__ __forceinline__ bool is_ws(unsigned char c) {
    return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

struct IsTerm {
    const unsigned char *buf;
    bool cr;
    __device__ int operator()(long long i) const { return is_term(buf[i], cr) ? 0 : -1; }
};
struct EmitIdx {
    __device__ long long operator()(long long i) const { return i; }
};

// line l spans [line_begin(l), line_end(l))
struct Lines {
    const unsigned char *buf;
    const long long *term;  // terminator positions, ascending
    long long nterm, nbytes;
    __device__ long long begin(long long l) const { return l == 0 ? 0 : term[l - 1] + 1; }
    __device__ long long end(long long l) const { return l < nterm ? term[l] : nbytes; }
};

struct IsEntry {
    Lines L;
    __device__ int operator()(long long l) const {
        const long long e = L.end(l);
        for (long long i = L.begin(l); i < e; ++i) {
            const unsigned char c = L.buf[i];
            if (is_ws(c)) continue;
            return c == '%' ? -1 : 0;  // comment line, or an entry
        }
        return -1;  // blank
    }
};

// Python int() over an ASCII token: [+-] digit (_? digit)*.  Saturates far
// above any node count (then the bounds check fails, as for the exact value).
__device__ bool parse_int(const unsigned char *s, long long len, long long &v) {
    long long i = 0;
    bool neg = false;
    if (len > 0 && (s[0] == '+' || s[0] == '-')) {
        neg = s[0] == '-';
        i = 1;
    }
    if (i >= len) return false;
    unsigned long long acc = 0;
    bool prev_us = true;  // no leading underscore
    constexpr unsigned long long SAT = 1ull << 62;
    for (; i < len; ++i) {
        const unsigned char c = s[i];
        if (c == '_') {
            if (prev_us) return false;
            prev_us = true;
            continue;
        }
        if (c < '0' || c > '9') return false;
        prev_us = false;
        if (acc < SAT / 16) acc = acc * 10 + (c - '0');
        else acc = SAT;
    }
    if (prev_us) return false;  // trailing underscore
    v = neg ? -(long long)acc : (long long)acc;
    return true;
}

__global__ void parse_entries_kernel(Lines L, const long long *entry_lines, long long nentries, long long rows,
                                     long long cols, long long nnz, long long *edges,
                                     unsigned long long *first_err) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nentries;
         k += (long long)gridDim.x * blockDim.x) {
        const long long l = entry_lines[k];
        const long long b = L.begin(l), e = L.end(l);
        long long tok[2][2];
        int nf = 0;
        long long i = b;
        while (nf < 2) {
            while (i < e && is_ws(L.buf[i])) ++i;
            if (i >= e) break;
            const long long t0 = i;
            while (i < e && !is_ws(L.buf[i])) ++i;
            tok[nf][0] = t0;
            tok[nf][1] = i;
            ++nf;
        }
        int code = 0;
        long long r = 0, c = 0;
        if (nf < 2) {
            code = HC_MTX_FEW_FIELDS;
        } else if (!parse_int(L.buf + tok[0][0], tok[0][1] - tok[0][0], r) ||
                   !parse_int(L.buf + tok[1][0], tok[1][1] - tok[1][0], c)) {
            code = HC_MTX_NON_INTEGER;
        } else if (!(1 <= r && r <= rows && 1 <= c && c <= cols)) {
            code = HC_MTX_BOUNDS;
        } else if (k >= nnz) {
            code = HC_MTX_TOO_MANY;
        }
        if (code) {
            atomicMin(first_err, ((unsigned long long)l << 3) | (unsigned long long)code);
        } else {
            edges[2 * k] = r - 1;
            edges[2 * k + 1] = c - 1;
        }
    }
}

__global__ void first_nonascii_kernel(const unsigned char *buf, long long n, unsigned long long *pos) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (buf[i] >= 0x80) atomicMin(pos, (unsigned long long)i);
}

// ------------------------------------------------------------------ degrees
constexpr int DS_THREADS = 512;
struct DegState {
    unsigned long long prefix;  // selected high digits so far
    unsigned long long k;       // rank still to find inside the selected bucket
    unsigned long long dmin, dmax;
};

// histogram of digit (deg >> shift) & (2^bits - 1) among degrees whose bits
// above shift+bits equal st->prefix; pass 0 also takes min / max
template <int BITS>
__global__ void __launch_bounds__(DS_THREADS) degree_hist_kernel(const long long *ro, long long n, int shift,
                                                                 DegState *st, unsigned long long *hist,
                                                                 bool first) {
    __shared__ unsigned h[1 << BITS];
    for (int i = threadIdx.x; i < (1 << BITS); i += DS_THREADS) h[i] = 0;
    __syncthreads();
    const unsigned long long pre = st->prefix;
    unsigned long long lo = ~0ull, hi = 0;
    for (long long u = (long long)blockIdx.x * DS_THREADS + threadIdx.x; u < n; u += (long long)gridDim.x * DS_THREADS) {
        const unsigned long long d = (unsigned long long)(ro[u + 1] - ro[u]);
        if (first) {
            lo = min(lo, d);
            hi = max(hi, d);
        }
        if ((d >> (shift + BITS)) == pre) atomicAdd(&h[(d >> shift) & ((1u << BITS) - 1u)], 1u);
    }
    if (first) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(FULL, lo, o));
            hi = max(hi, __shfl_xor_sync(FULL, hi, o));
        }
        if (lane_id() == 0) {
            atomicMin(&st->dmin, lo);
            atomicMax(&st->dmax, hi);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (1 << BITS); i += DS_THREADS)
        if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

// one CTA: bucket holding rank st->k; append its digit to the prefix and
// clear the histogram for the next pass
template <int BITS>
__global__ void __launch_bounds__(1024) degree_select_kernel(DegState *st, unsigned long long *hist) {
    constexpr int NBK = 1 << BITS;
    constexpr int PER = (NBK + 1023) / 1024;
    __shared__ unsigned long long warp_tot[32];
    __shared__ unsigned long long s_base;
    unsigned long long v[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int i = threadIdx.x * PER + q;
        v[q] = i < NBK ? hist[i] : 0ull;
        sum += v[q];
    }
    const unsigned long long incl = warp_incl_scan(sum);
    if (lane_id() == 31) warp_tot[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        const unsigned long long w = warp_tot[threadIdx.x];
        const unsigned long long wi = warp_incl_scan(w);
        warp_tot[threadIdx.x] = wi - w;
    }
    __syncthreads();
    unsigned long long run = warp_tot[threadIdx.x >> 5] + incl - sum;  // elements before my first bucket
    const unsigned long long k = st->k;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int i = threadIdx.x * PER + q;
        if (i < NBK && run <= k && k < run + v[q]) {  // exactly one thread matches
            st->prefix = (st->prefix << BITS) | (unsigned long long)i;
            s_base = run;
        }
        run += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) st->k = k - s_base;
    for (int i = threadIdx.x; i < NBK; i += 1024) hist[i] = 0;
}

}  // namespace ingest
}  // namespace hcb

using namespace hcb;
using namespace hcb::ingest;

extern "C" {

size_t hc_mtx_workspace_bytes(int64_t num_bytes) {
    const long long n = num_bytes < 0 ? 0 : num_bytes;
    // terminator positions + entry-line ids (each <= n + 1 int64) + partition
    // scratch + two u64 results
    return align_up(8 * (size_t)(n + 1), 256) * 2 + part_scratch_bytes(1, n + 1) + 256;
}

int hc_mtx_parse(const uint8_t *d_bytes, int64_t num_bytes, int universal_newlines, int64_t rows, int64_t cols,
                 int64_t nnz, int64_t *d_edges, int64_t *h_num_entries, int64_t *h_err_line, int *h_err_code,
                 int64_t *h_err_span, int64_t *h_first_nonascii, void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(num_bytes >= 0 && rows >= 0 && cols >= 0 && nnz >= 0, HC_ERR_INVALID, "hc_mtx_parse: bad sizes");
    HC_REQUIRE(h_num_entries && h_err_line && h_err_code && h_err_span && h_first_nonascii, HC_ERR_INVALID,
               "hc_mtx_parse: null output pointer");
    HC_REQUIRE((num_bytes == 0 || d_bytes) && (nnz == 0 || d_edges), HC_ERR_INVALID, "hc_mtx_parse: null buffer");
    HC_REQUIRE(d_ws && ws_bytes >= hc_mtx_workspace_bytes(num_bytes), HC_ERR_WORKSPACE,
               "hc_mtx_parse: workspace too small");
    cudaStream_t st = as_stream(stream);
    *h_num_entries = 0;
    *h_err_line = -1;
    *h_err_code = 0;
    *h_first_nonascii = -1;
    const long long n = num_bytes;
    char *ws = reinterpret_cast<char *>(d_ws);
    long long *term = reinterpret_cast<long long *>(ws);
    long long *entries = reinterpret_cast<long long *>(ws + align_up(8 * (size_t)(n + 1), 256));
    char *scratch = ws + 2 * align_up(8 * (size_t)(n + 1), 256);
    unsigned long long *res = reinterpret_cast<unsigned long long *>(scratch + part_scratch_bytes(1, n + 1));
    HC_CUDA_TRY(cudaMemsetAsync(res, 0xff, 2 * sizeof(unsigned long long), st));
    const int sms = std::max(1, num_sms());
    if (n > 0) {
        first_nonascii_kernel<<<sms * 8, 256, 0, st>>>(d_bytes, n, res + 1);
        HC_CHECK_LAUNCH();
    }
    unsigned long long *tot = nullptr;
    int rc = ordered_partition<1>(n, IsTerm{d_bytes, universal_newlines != 0}, EmitIdx{}, term, scratch, &tot, st);
    if (rc != HC_OK) return rc;
    unsigned long long nterm = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&nterm, tot, 8, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    const long long nlines = (long long)nterm + 1;
    Lines L{d_bytes, term, (long long)nterm, n};
    rc = ordered_partition<1>(nlines, IsEntry{L}, EmitIdx{}, entries, scratch, &tot, st);
    if (rc != HC_OK) return rc;
    unsigned long long nent = 0;
    HC_CUDA_TRY(cudaMemcpyAsync(&nent, tot, 8, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    if (nent > 0) {
        const long long blocks = std::min<long long>(((long long)nent + 255) / 256, (long long)sms * 32);
        parse_entries_kernel<<<(unsigned)blocks, 256, 0, st>>>(L, entries, (long long)nent, rows, cols, nnz, (long long *)d_edges,
                                                               res);
        HC_CHECK_LAUNCH();
    }
    unsigned long long h_res[2];
    HC_CUDA_TRY(cudaMemcpyAsync(h_res, res, sizeof h_res, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    *h_num_entries = (int64_t)nent;
    if (h_res[0] != ~0ull) {  // the offending line and its byte span [begin, end)
        const long long l = (long long)(h_res[0] >> 3);
        *h_err_line = l;
        *h_err_code = (int)(h_res[0] & 7ull);
        long long b = -1, e = n;
        if (l > 0) HC_CUDA_TRY(cudaMemcpyAsync(&b, term + l - 1, 8, cudaMemcpyDeviceToHost, st));
        if (l < (long long)nterm) HC_CUDA_TRY(cudaMemcpyAsync(&e, term + l, 8, cudaMemcpyDeviceToHost, st));
        HC_CUDA_TRY(cudaStreamSynchronize(st));
        h_err_span[0] = b + 1;
        h_err_span[1] = e;
    }
    if (h_res[1] != ~0ull) *h_first_nonascii = (int64_t)h_res[1];
    return HC_OK;
}

size_t hc_degree_stats_workspace_bytes(void) {
    return align_up(sizeof(DegState), 256) + sizeof(unsigned long long) * 2048;
}

int hc_degree_stats(const int64_t *d_row_offsets, int64_t num_nodes, int64_t *h_min, int64_t *h_median,
                    int64_t *h_max, void *d_ws, size_t ws_bytes, void *stream) {
    HC_REQUIRE(num_nodes > 0, HC_ERR_INVALID, "degree statistics are undefined for an empty graph");
    HC_REQUIRE(d_row_offsets && h_min && h_median && h_max, HC_ERR_INVALID, "hc_degree_stats: null pointer");
    HC_REQUIRE(d_ws && ws_bytes >= hc_degree_stats_workspace_bytes(), HC_ERR_WORKSPACE,
               "hc_degree_stats: workspace too small");
    cudaStream_t st = as_stream(stream);
    DegState *S = reinterpret_cast<DegState *>(d_ws);
    unsigned long long *hist = reinterpret_cast<unsigned long long *>((char *)d_ws + align_up(sizeof(DegState), 256));
    DegState init{0ull, (unsigned long long)(num_nodes / 2), ~0ull, 0ull};
    HC_CUDA_TRY(cudaMemcpyAsync(S, &init, sizeof init, cudaMemcpyHostToDevice, st));
    HC_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 2048, st));
    const long long *ro = reinterpret_cast<const long long *>(d_row_offsets);
    const unsigned blocks = (unsigned)std::min<long long>((num_nodes + DS_THREADS - 1) / DS_THREADS,
                                                          (long long)std::max(1, num_sms()) * 4);
    // degrees < 2^31: digits [30..20] (11 bits), [19..9] (11), [8..0] (9)
    degree_hist_kernel<11><<<blocks, DS_THREADS, 0, st>>>(ro, num_nodes, 20, S, hist, true);
    HC_CHECK_LAUNCH();
    degree_select_kernel<11><<<1, 1024, 0, st>>>(S, hist);
    HC_CHECK_LAUNCH();
    degree_hist_kernel<11><<<blocks, DS_THREADS, 0, st>>>(ro, num_nodes, 9, S, hist, false);
    HC_CHECK_LAUNCH();
    degree_select_kernel<11><<<1, 1024, 0, st>>>(S, hist);
    HC_CHECK_LAUNCH();
    degree_hist_kernel<9><<<blocks, DS_THREADS, 0, st>>>(ro, num_nodes, 0, S, hist, false);
    HC_CHECK_LAUNCH();
    degree_select_kernel<9><<<1, 1024, 0, st>>>(S, hist);
    HC_CHECK_LAUNCH();
    DegState out;
    HC_CUDA_TRY(cudaMemcpyAsync(&out, S, sizeof out, cudaMemcpyDeviceToHost, st));
    HC_CUDA_TRY(cudaStreamSynchronize(st));
    *h_min = (int64_t)out.dmin;
    *h_max = (int64_t)out.dmax;
    *h_median = (int64_t)out.prefix;
    return HC_OK;
}

}  // extern "C"
