// Hardware counters by human-readable name for xtc_measure (the
// paper's counter path: "retrieves hardware counters by name",
// P:833-837 "CUPTI ... gpu. prefix"). One CUPTI range-profiler range (user range,
// user replay) is wrapped around one call of the operator, in a pass of its own
// after the timed reps: multi-pass metrics are replayed by re-running the call, which
// is idempotent (every output element is rewritten). CUPTI is dlopen'ed here so that
// libxtc.so loads on machines without it; a missing library or an unsupported
// device/metric is reported as "unavailable", never as a failed measurement.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "xtc_internal.h"

namespace xtc {
namespace {

#define CUPTI_FNS(X)                                 \
    X(cuptiProfilerInitialize)                       \
    X(cuptiProfilerDeInitialize)                     \
    X(cuptiDeviceGetChipName)                        \
    X(cuptiProfilerGetCounterAvailability)           \
    X(cuptiProfilerHostInitialize)                   \
    X(cuptiProfilerHostDeinitialize)                 \
    X(cuptiProfilerHostConfigAddMetrics)             \
    X(cuptiProfilerHostGetConfigImageSize)           \
    X(cuptiProfilerHostGetConfigImage)               \
    X(cuptiProfilerHostEvaluateToGpuValues)          \
    X(cuptiRangeProfilerEnable)                      \
    X(cuptiRangeProfilerDisable)                     \
    X(cuptiRangeProfilerGetCounterDataSize)          \
    X(cuptiRangeProfilerCounterDataImageInitialize)  \
    X(cuptiRangeProfilerSetConfig)                   \
    X(cuptiRangeProfilerStart)                       \
    X(cuptiRangeProfilerStop)                        \
    X(cuptiRangeProfilerPushRange)                   \
    X(cuptiRangeProfilerPopRange)                    \
    X(cuptiRangeProfilerDecodeData)

struct Cupti {
#define DECL(f) decltype(&::f) f = nullptr;
    CUPTI_FNS(DECL)
#undef DECL
    const char* (*get_result_string)(CUptiResult, const char**) = nullptr;
    bool ok = false;
    std::string why;
};

Cupti& cupti() {
    static Cupti c;
    static std::once_flag once;
    std::call_once(once, [] {
        // libnvperf_host is opened by CUPTI by soname: load it first, globally, from the
        // toolkit so the soname resolves without LD_LIBRARY_PATH
        const char* perf[] = {"libnvperf_host.so", "/usr/local/cuda/lib64/libnvperf_host.so",
                              "/usr/local/cuda/extras/CUPTI/lib64/libnvperf_host.so"};
        for (const char* p : perf)
            if (dlopen(p, RTLD_NOW | RTLD_GLOBAL)) break;
        const char* names[] = {"libcupti.so.12", "/usr/local/cuda/lib64/libcupti.so.12",
                               "/usr/local/cuda/extras/CUPTI/lib64/libcupti.so.12", "libcupti.so"};
        void* h = nullptr;
        for (const char* n : names)
            if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            c.why = "libcupti.so.12 not found";
            return;
        }
#define LOAD(f)                                                              \
    c.f = reinterpret_cast<decltype(&::f)>(dlsym(h, #f));                    \
    if (!c.f) {                                                              \
        c.why = "libcupti lacks " #f;                                        \
        return;                                                              \
    }
        CUPTI_FNS(LOAD)
#undef LOAD
        c.get_result_string = reinterpret_cast<const char* (*)(CUptiResult, const char**)>(
            dlsym(h, "cuptiGetResultString"));
        c.ok = true;
    });
    return c;
}

std::string cupti_err(const char* what, CUptiResult r) {
    const char* s = nullptr;
    if (cupti().get_result_string) cupti().get_result_string(r, &s);
    return std::string(what) + ": " + (s ? s : "CUPTI error " + std::to_string((int)r));
}

}  // namespace

std::vector<std::string> split_counter_names(const char* list) {
    std::vector<std::string> out;
    if (!list) return out;
    std::string cur;
    auto flush = [&] {
        size_t a = cur.find_first_not_of(" \t"), b = cur.find_last_not_of(" \t");
        std::string n = a == std::string::npos ? "" : cur.substr(a, b - a + 1);
        if (n.rfind("gpu.", 0) == 0) n = n.substr(4);  // "gpu." names a hardware counter
        if (!n.empty()) out.push_back(n);
        cur.clear();
    };
    for (const char* p = list; *p; ++p) {
        if (*p == ',') flush();
        else cur.push_back(*p);
    }
    flush();
    return out;
}

bool collect_counters(int device, const std::vector<std::string>& names, const std::function<bool()>& prepare,
                      const std::function<bool()>& run_once, std::vector<double>& values, std::string& why) {
    Cupti& c = cupti();
    if (!c.ok) {
        why = c.why;
        return false;
    }
    static std::mutex mu;  // one profiling session per process at a time
    std::lock_guard<std::mutex> lock(mu);

    CUcontext ctx = nullptr;
    {
        using GetCur = CUresult (*)(CUcontext*);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
            reinterpret_cast<GetCur>(fn)(&ctx) != CUDA_SUCCESS || !ctx) {
            why = "no current CUDA context";
            return false;
        }
    }
    CUptiResult r;
#define CK(call, what)                       \
    if ((r = (call)) != CUPTI_SUCCESS) {     \
        why = cupti_err(what, r);            \
        goto done;                           \
    }
    std::vector<const char*> pn;
    for (const auto& n : names) pn.push_back(n.c_str());
    std::vector<uint8_t> avail, config, data;
    CUpti_Profiler_Host_Object* host = nullptr;
    CUpti_RangeProfiler_Object* obj = nullptr;
    bool ok = false;
    {
        CUpti_Profiler_Initialize_Params ip{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
        CK(c.cuptiProfilerInitialize(&ip), "cuptiProfilerInitialize");
    }
    {
        CUpti_Device_GetChipName_Params cp{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
        cp.deviceIndex = (size_t)device;
        CK(c.cuptiDeviceGetChipName(&cp), "cuptiDeviceGetChipName");
        CUpti_Profiler_GetCounterAvailability_Params ap{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
        ap.ctx = ctx;
        CK(c.cuptiProfilerGetCounterAvailability(&ap), "counter availability size");
        avail.resize(ap.counterAvailabilityImageSize);
        ap.pCounterAvailabilityImage = avail.data();
        CK(c.cuptiProfilerGetCounterAvailability(&ap), "counter availability");

        CUpti_Profiler_Host_Initialize_Params hp{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
        hp.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
        hp.pChipName = cp.pChipName;
        hp.pCounterAvailabilityImage = avail.data();
        CK(c.cuptiProfilerHostInitialize(&hp), "cuptiProfilerHostInitialize");
        host = hp.pHostObject;
    }
    {
        CUpti_Profiler_Host_ConfigAddMetrics_Params mp{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
        mp.pHostObject = host;
        mp.ppMetricNames = pn.data();
        mp.numMetrics = pn.size();
        CK(c.cuptiProfilerHostConfigAddMetrics(&mp), "unknown metric name");
        CUpti_Profiler_Host_GetConfigImageSize_Params sp{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
        sp.pHostObject = host;
        CK(c.cuptiProfilerHostGetConfigImageSize(&sp), "config image size");
        config.resize(sp.configImageSize);
        CUpti_Profiler_Host_GetConfigImage_Params gp{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
        gp.pHostObject = host;
        gp.pConfigImage = config.data();
        gp.configImageSize = config.size();
        CK(c.cuptiProfilerHostGetConfigImage(&gp), "config image");
    }
    {
        CUpti_RangeProfiler_Enable_Params ep{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
        ep.ctx = ctx;
        CK(c.cuptiRangeProfilerEnable(&ep), "cuptiRangeProfilerEnable");
        obj = ep.pRangeProfilerObject;

        CUpti_RangeProfiler_GetCounterDataSize_Params dp{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
        dp.pRangeProfilerObject = obj;
        dp.pMetricNames = pn.data();
        dp.numMetrics = pn.size();
        dp.maxNumOfRanges = 1;
        dp.maxNumRangeTreeNodes = 1;
        CK(c.cuptiRangeProfilerGetCounterDataSize(&dp), "counter data size");
        data.resize(dp.counterDataSize);
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params ip{
            CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
        ip.pRangeProfilerObject = obj;
        ip.counterDataSize = data.size();
        ip.pCounterData = data.data();
        CK(c.cuptiRangeProfilerCounterDataImageInitialize(&ip), "counter data init");

        CUpti_RangeProfiler_SetConfig_Params cp{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
        cp.pRangeProfilerObject = obj;
        cp.configSize = config.size();
        cp.pConfig = config.data();
        cp.counterDataImageSize = data.size();
        cp.pCounterDataImage = data.data();
        cp.range = CUPTI_UserRange;
        cp.replayMode = CUPTI_UserReplay;
        cp.maxRangesPerPass = 1;
        cp.numNestingLevels = 1;
        cp.minNestingLevel = 1;
        cp.passIndex = 0;
        cp.targetNestingLevel = 1;
        CK(c.cuptiRangeProfilerSetConfig(&cp), "cuptiRangeProfilerSetConfig");
    }
    for (int pass = 0;; ++pass) {
        if (pass >= 256) {
            why = "more than 256 replay passes";
            goto done;
        }
        if (!prepare()) {  // outside the range: e.g. the L2 flush before every replay
            why = "prepare step failed during counter replay";
            goto done;
        }
        CUpti_RangeProfiler_Start_Params sp{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
        sp.pRangeProfilerObject = obj;
        CK(c.cuptiRangeProfilerStart(&sp), "cuptiRangeProfilerStart");
        CUpti_RangeProfiler_PushRange_Params pp{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
        pp.pRangeProfilerObject = obj;
        pp.pRangeName = "xtc_run";
        CK(c.cuptiRangeProfilerPushRange(&pp), "cuptiRangeProfilerPushRange");
        if (!run_once()) {
            why = "operator call failed during counter replay";
            goto done;
        }
        CUpti_RangeProfiler_PopRange_Params qp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
        qp.pRangeProfilerObject = obj;
        CK(c.cuptiRangeProfilerPopRange(&qp), "cuptiRangeProfilerPopRange");
        CUpti_RangeProfiler_Stop_Params tp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
        tp.pRangeProfilerObject = obj;
        CK(c.cuptiRangeProfilerStop(&tp), "cuptiRangeProfilerStop");
        if (tp.isAllPassSubmitted) break;
    }
    {
        CUpti_RangeProfiler_DecodeData_Params dp{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
        dp.pRangeProfilerObject = obj;
        CK(c.cuptiRangeProfilerDecodeData(&dp), "cuptiRangeProfilerDecodeData");
        values.assign(names.size(), 0.0);
        CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
        ev.pHostObject = host;
        ev.pCounterDataImage = data.data();
        ev.counterDataImageSize = data.size();
        ev.rangeIndex = 0;
        ev.ppMetricNames = pn.data();
        ev.numMetrics = pn.size();
        ev.pMetricValues = values.data();
        CK(c.cuptiProfilerHostEvaluateToGpuValues(&ev), "cuptiProfilerHostEvaluateToGpuValues");
        ok = true;
    }
done:
#undef CK
    if (obj) {
        CUpti_RangeProfiler_Disable_Params dp{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        dp.pRangeProfilerObject = obj;
        c.cuptiRangeProfilerDisable(&dp);
    }
    if (host) {
        CUpti_Profiler_Host_Deinitialize_Params hp{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
        hp.pHostObject = host;
        c.cuptiProfilerHostDeinitialize(&hp);
    }
    return ok;
}

}  // namespace xtc
