// prof.cu — event-pair recorder behind prof.cuh and its C ABI.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/helr_ckks.h"
#include "ctx.cuh"
#include "prof.cuh"

namespace {
struct Rec {
    int cat;
    double bytes;
    cudaEvent_t a, b;
};
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
int g_open = -1;

cudaEvent_t take() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

bool prof_enabled() { return g_on; }

static unsigned long long g_launches = 0;
void count_launches(int k) { g_launches += (unsigned long long)k; }
extern "C" unsigned long long helr_launch_count(void) { return g_launches; }

bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HELR_PDL");
        on = e ? (atoi(e) != 0) : 1;
    }
    return on != 0;
}

// single-pass cluster NTT for N = 2^16 (ntt_cluster.cuh): HELR_NTT_CLUSTER=0
// falls back to the two-pass kernels; HELR_NTT_CL_MIN = fewest limb
// transforms per launch that take the cluster path
bool ntt_cluster_enabled(long long limb_transforms) {
    static int on = -1;
    static long long lo = 1, hi = 1ll << 40;
    if (on < 0) {
        const char* e = getenv("HELR_NTT_CLUSTER");
        on = e ? (atoi(e) != 0) : 0;  // measured slower than the two-pass kernels
        const char* m = getenv("HELR_NTT_CL_MIN");
        lo = m ? atoll(m) : 1;
        const char* x = getenv("HELR_NTT_CL_MAX");  // e.g. only the small single-ciphertext launches
        hi = x ? atoll(x) : (1ll << 40);
    }
    return on != 0 && limb_transforms >= lo && limb_transforms <= hi;
}
// cp.async.bulk for the dense tile of the cluster NTT (HELR_NTT_BULK=0: plain loads / stores)
bool ntt_bulk_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HELR_NTT_BULK");
        on = e ? (atoi(e) != 0) : 1;
    }
    return on != 0;
}

// cluster NTT exchange through st.async + mbarrier (HELR_NTT_XASYNC=0: cluster barriers)
bool ntt_xasync_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("HELR_NTT_XASYNC");
        on = e ? (atoi(e) != 0) : 1;
    }
    return on != 0;
}

// external event nodes inside a graph capture, plain records otherwise
static cudaError_t record(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) cudaGetLastError();
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                               : cudaEventRecord(ev, s);
}

void prof_begin(int cat, double bytes, cudaStream_t s) {
    Rec r{cat, bytes, take(), take()};
    cudaError_t e = record(r.a, s);
    if (e != cudaSuccess) {
        fprintf(stderr, "[helr prof] cudaEventRecord(begin) failed: %s\n", cudaGetErrorString(e));
        cudaGetLastError();
        return;
    }
    g_recs.push_back(r);
    g_open = (int)g_recs.size() - 1;
}

void prof_end(cudaStream_t s) {
    if (g_open < 0) return;
    cudaError_t e = record(g_recs[g_open].b, s);
    if (e != cudaSuccess) {
        fprintf(stderr, "[helr prof] cudaEventRecord(end) failed: %s\n", cudaGetErrorString(e));
        cudaGetLastError();
        g_recs.pop_back();
    }
    g_open = -1;
}

extern "C" int helr_prof_enable(int on) {
    g_on = on != 0;
    return HELR_OK;
}

// Synchronises, then fills per-category totals: ms[cat], bytes[cat],
// launches[cat] (arrays of HELR_PROF_NCAT) and clears the record list.
extern "C" int helr_prof_collect(double* ms, double* bytes, int* launches) {
    if (!cuda_ok(cudaDeviceSynchronize(), "prof sync")) return HELR_ECUDA;
    for (int c = 0; c < PROF_NCAT; c++) { ms[c] = 0; bytes[c] = 0; launches[c] = 0; }
    for (auto& r : g_recs) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) { cudaGetLastError(); t = 0.f; }
        ms[r.cat] += t;
        bytes[r.cat] += r.bytes;
        launches[r.cat] += 1;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    return HELR_OK;
}
