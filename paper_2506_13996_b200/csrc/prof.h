// Per-kernel-class CUDA-event timing inside the timed region (bench roofline evidence).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <sstream>
#include <string>
#include <vector>

#include "common.h"
#include "launch.h"

namespace spt {

// ---------------------------------------------------------------- per-kernel-class event timing
struct Prof {
    bool on = false;
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        double flops, bytes;
        int64_t launches;
        std::string tag;  // optional finer key (e.g. GEMM shape/epilogue) for the per-site breakdown
    };
    std::string next_tag;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    static constexpr int NCLS = 9;
    static const char* name(int c) {
        static const char* n[] = {"gemm", "attn_fwd", "attn_bwd", "rmsnorm", "reshard", "ce_rows", "comm", "other",
                                  "a2a"};
        return n[c];
    }
    cudaEvent_t ev() {
        if (used == pool.size()) {
            cudaEvent_t e;
            SPT_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    void reset() {
        recs.clear();
        used = 0;
    }
    template <class F>
    void run(int cls, double flops, double bytes, cudaStream_t st, F&& f) {
        if (!on) {
            f();
            return;
        }
        cudaEvent_t a = ev(), b = ev();
        const int64_t n0 = launch_count();
        // External records: under stream capture they become event-record nodes of the graph, re-recorded by every
        // replay, so the per-class times of a replayed step are readable afterwards (bench.py times its graph
        // replays with profiling on: the roofline comes from inside the timed region).
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        SPT_CUDA(cudaStreamIsCapturing(st, &cs));
        const unsigned fl = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
        SPT_CUDA(cudaEventRecordWithFlags(a, st, fl));
        f();
        SPT_CUDA(cudaEventRecordWithFlags(b, st, fl));
        recs.push_back({cls, a, b, flops, bytes, launch_count() - n0, next_tag});
        next_tag.clear();
    }
    // Time between consecutive profiled regions of the last step (unprofiled kernels, launch gaps, kernel ramp-up
    // outside the events): total and the largest few, keyed "<class before>-><class after>#<record index>".
    std::string gaps_json() {
        std::ostringstream os;
        double gap_total = 0;
        std::vector<std::pair<double, std::string>> gaps;
        for (size_t i = 1; i < recs.size(); ++i) {
            float t = 0;
            if (cudaEventElapsedTime(&t, recs[i - 1].b, recs[i].a) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (t <= 0) continue;
            gap_total += t;
            gaps.push_back({t, std::string(name(recs[i - 1].cls)) + "->" + name(recs[i].cls) + "#" + std::to_string(i)});
        }
        std::sort(gaps.begin(), gaps.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
        os << "{\"ms\":" << gap_total << ",\"n\":" << gaps.size() << ",\"top\":{";
        for (size_t i = 0; i < gaps.size() && i < 6; ++i)
            os << (i ? "," : "") << "\"" << gaps[i].second << "\":" << gaps[i].first;
        os << "}}";
        return os.str();
    }
    std::string json() {
        double ms[NCLS] = {}, fl[NCLS] = {}, by[NCLS] = {};
        int cnt[NCLS] = {};
        for (auto& r : recs) {
            float t = 0;
            SPT_CUDA(cudaEventSynchronize(r.b));
            SPT_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            ms[r.cls] += t;
            fl[r.cls] += r.flops;
            by[r.cls] += r.bytes;
            cnt[r.cls] += (int)r.launches;
        }
        std::ostringstream os;
        // per-tag breakdown (GEMM call sites)
        std::vector<std::string> tags;
        std::vector<double> tms, tfl, tby;
        std::vector<int> tn;
        for (auto& r : recs) {
            if (r.tag.empty()) continue;
            float t = 0;
            SPT_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            size_t i = 0;
            while (i < tags.size() && tags[i] != r.tag) ++i;
            if (i == tags.size()) {
                tags.push_back(r.tag);
                tms.push_back(0);
                tfl.push_back(0);
                tby.push_back(0);
                tn.push_back(0);
            }
            tms[i] += t;
            tfl[i] += r.flops;
            tby[i] += r.bytes;
            tn[i] += 1;
        }
        os << "{\"sites\":{";
        for (size_t i = 0; i < tags.size(); ++i)
            os << (i ? "," : "") << "\"" << tags[i] << "\":{\"ms\":" << tms[i] << ",\"calls\":" << tn[i]
               << ",\"tflops\":" << (tms[i] > 0 ? tfl[i] / (tms[i] * 1e9) : 0)
               << ",\"bytes\":" << tby[i] << ",\"gbps\":" << (tms[i] > 0 ? tby[i] / (tms[i] * 1e6) : 0) << "}";
        os << "},";
        for (int c = 0; c < NCLS; ++c)
            os << (c ? "," : "") << "\"" << name(c) << "\":{\"ms\":" << ms[c] << ",\"launches\":" << cnt[c]
               << ",\"flops\":" << fl[c] << ",\"bytes\":" << by[c] << "}";
        os << "}";
        return os.str();
    }
};
// P_A2A: a Ulysses all-to-all with its pack / unpack kernel fused in (bytes = payload sent to peers)
enum { P_GEMM = 0, P_ATTN_F, P_ATTN_B, P_NORM, P_RESHARD, P_CE, P_COMM, P_OTHER, P_A2A };

// The engine installs its Prof here for the duration of a step; library launchers (gemm, ce_rows)
// self-report so multi-kernel helpers (flce, mlp) are attributed per kernel class.
Prof*& current_prof();

template <class F>
inline void prof_run(int cls, double flops, double bytes, cudaStream_t st, F&& f) {
    Prof* p = current_prof();
    if (p && p->on) p->run(cls, flops, bytes, st, f);
    else f();
}

}  // namespace spt
