// Launch accounting and per-kernel CUDA-event tracing.
//
// Every kernel the library launches goes through NSM_PROF(name, stream):
// a process-wide launch counter (the bench's `gpu_launches`) and, when
// tracing is on (nsm_profile_enable), a pair of CUDA events recorded on the
// launching stream around the launch.  nsm_profile_report synchronises the
// recorded events and returns per-kernel launch counts and average device
// durations -- the live per-kernel timing the roofline figure uses.
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "prof.cuh"

namespace nsm {

namespace {
std::atomic<long long> g_launches{0};
std::atomic<int> g_enabled{0};
std::mutex g_mu;
struct Rec {
    std::string name;
    cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

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

ProfScope::ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_enabled.load(std::memory_order_relaxed)) return;
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    std::lock_guard<std::mutex> lk(g_mu);
    a_ = take();
    b_ = take();
    cudaEventRecord(a_, s);
    on_ = true;
}

ProfScope::~ProfScope() {
    if (!on_) return;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaEventRecord(b_, s_);
    g_recs.push_back({name_, a_, b_});
}

}  // namespace nsm

using namespace nsm;

extern "C" {

int64_t nsm_launch_count(void) { return g_launches.load(); }

void nsm_profile_enable(int32_t on) { g_enabled.store(on ? 1 : 0); }

int32_t nsm_profile_report(char* buf, size_t cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, std::pair<long long, double>> agg;
    for (auto& r : g_recs) {
        cudaEventSynchronize(r.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& v = agg[r.name];
        v.first += 1;
        v.second += ms;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    std::string out;
    for (auto& kv : agg) {
        char line[256];
        snprintf(line, sizeof line, "%s %lld %.6f\n", kv.first.c_str(), kv.second.first,
                 kv.second.second);
        out += line;
    }
    if (buf && cap) {
        size_t n = std::min(cap - 1, out.size());
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return (int32_t)out.size();
}

}  // extern "C"
