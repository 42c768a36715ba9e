// hcb_common.cu -- error reporting, device queries and the partition scan.
#include <mutex>
#include <string>

#include "hcb_partition.cuh"

namespace hcb {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

int num_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return sms;
}

__global__ void __launch_bounds__(PART_SCAN_THREADS) part_scan_kernel(unsigned long long *vals,
                                                                      long long len, int nb,
                                                                      long long tiles,
                                                                      unsigned long long *totals) {
    __shared__ unsigned long long s_warp[PART_SCAN_THREADS / 32];
    __shared__ unsigned long long s_total;
    const long long per = (len + PART_SCAN_THREADS - 1) / PART_SCAN_THREADS;
    const long long lo = min(len, per * threadIdx.x), hi = min(len, lo + per);
    unsigned long long local = 0;
    for (long long i = lo; i < hi; ++i) local += vals[i];
    unsigned long long incl = warp_incl_scan(local);
    const unsigned warp = threadIdx.x >> 5;
    if (lane_id() == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long v = s_warp[lane_id()];
        unsigned long long vi = warp_incl_scan(v);
        s_warp[lane_id()] = vi - v;
        if (lane_id() == 31) s_total = vi;
    }
    __syncthreads();
    unsigned long long run = incl - local + s_warp[warp];
    for (long long i = lo; i < hi; ++i) {
        unsigned long long v = vals[i];
        vals[i] = run;
        run += v;
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)nb) {
        const int b = threadIdx.x;
        unsigned long long start = vals[(long long)b * tiles];
        unsigned long long end = (b + 1 < nb) ? vals[(long long)(b + 1) * tiles] : s_total;
        totals[b] = end - start;
    }
}

}  // namespace hcb

extern "C" {

const char *hc_last_error(void) { return hcb::g_last_error.c_str(); }

int hc_version(void) { return 1; }

}  // extern "C"
