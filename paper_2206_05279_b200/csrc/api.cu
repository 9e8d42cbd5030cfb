// Library identity and device check.
#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace {
const char *kCatNames[PROF_NCAT] = {"conv_kernel",        "argmin_kernel",  "rans_encode_kernel",
                                    "rans_decode_kernel", "twar_forward_kernel", "twar_decode_kernel",
                                    "static_scale_kernel", "blob_sizes+scan", "pack_kernel",
                                    "parse_kernel",       "lanes_kernel",   "crc_kernel",
                                    "sched_crc_kernel",   "tc_conv_kernel", "gather_kernel",
                                    "tc3_conv_kernel", "enc_front_kernel", "tc3_block_kernel", "dec_trunk_kernel", "enc_trunk_kernel",
                                    "dec_uphead_kernel", "dec_trunk2_kernel"};
struct Rec {
    int cat;
    cudaEvent_t e0, e1;
    double units;
};
std::atomic<long long> g_launches{0};
std::atomic<int> g_timing{0};
std::mutex g_mu;
std::vector<Rec> g_recs;
}  // namespace

void *prof_begin(int cat, cudaStream_t s, double units) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_timing.load(std::memory_order_relaxed)) return nullptr;
    Rec *r = new Rec{cat, nullptr, nullptr, units};
    cudaEventCreate(&r->e0);
    cudaEventCreate(&r->e1);
    cudaEventRecord(r->e0, s);
    return r;
}

void prof_end(void *tok, cudaStream_t s) {
    if (!tok) return;
    Rec *r = static_cast<Rec *>(tok);
    cudaEventRecord(r->e1, s);
    std::lock_guard<std::mutex> g(g_mu);
    g_recs.push_back(*r);
    delete r;
}

extern "C" void pilc_prof_reset(int32_t enable_timing) {
    std::lock_guard<std::mutex> g(g_mu);
    for (auto &r : g_recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    g_recs.clear();
    g_launches.store(0);
    g_timing.store(enable_timing ? 1 : 0);
}

extern "C" int64_t pilc_prof_launches(void) { return g_launches.load(); }

extern "C" int64_t pilc_prof_count(void) {
    std::lock_guard<std::mutex> g(g_mu);
    return (int64_t)g_recs.size();
}

extern "C" int pilc_prof_record(int64_t i, int32_t *cat, double *ms, double *units) {
    std::lock_guard<std::mutex> g(g_mu);
    if (i < 0 || i >= (int64_t)g_recs.size()) return PILC_E_ARG;
    const Rec &r = g_recs[(size_t)i];
    if (cudaEventSynchronize(r.e1) != cudaSuccess) return PILC_E_CUDA;
    float t = 0;
    cudaEventElapsedTime(&t, r.e0, r.e1);
    *cat = r.cat;
    *ms = t;
    *units = r.units;
    return PILC_OK;
}

extern "C" int32_t pilc_prof_categories(void) { return PROF_NCAT; }

extern "C" const char *pilc_prof_name(int32_t cat) {
    return (cat >= 0 && cat < PROF_NCAT) ? kCatNames[cat] : "";
}

extern "C" int pilc_prof_read(int32_t cat, int64_t *launches, double *total_ms, double *units) {
    if (cat < 0 || cat >= PROF_NCAT) return PILC_E_ARG;
    std::lock_guard<std::mutex> g(g_mu);
    int64_t n = 0;
    double ms = 0, u = 0;
    for (auto &r : g_recs) {
        if (r.cat != cat) continue;
        if (cudaEventSynchronize(r.e1) != cudaSuccess) return PILC_E_CUDA;
        float t = 0;
        cudaEventElapsedTime(&t, r.e0, r.e1);
        ++n;
        ms += t;
        u += r.units;
    }
    *launches = n;
    *total_ms = ms;
    *units = u;
    return PILC_OK;
}

int g_tuning[PILC_TUNE_N] = {1, 2, 1, 1};

extern "C" int pilc_set_tuning(int32_t key, int32_t value) {
    if (key < 0 || key >= PILC_TUNE_N) return -PILC_E_ARG;
    const int prev = g_tuning[key];
    g_tuning[key] = value;
    return prev;
}

extern "C" const char *pilc_version(void) { return "pilc-sm100a 0.1.0"; }

extern "C" int pilc_device_arch(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return p.major * 10 + p.minor;
}

int dyn_smem_limit(const void *func) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({func, dev});
    if (it != cache.end()) return it->second;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    int v = optin;
    if (cudaFuncGetAttributes(&fa, func) == cudaSuccess) v = optin - (int)fa.sharedSizeBytes;
    else cudaGetLastError();
    cache[{func, dev}] = v;
    return v;
}
