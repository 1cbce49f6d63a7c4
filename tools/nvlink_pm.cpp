// nvlink_pm.cpp — NVLink (and DRAM) bytes of one GPU over a time window, from CUPTI PM
// sampling (device-level hardware counters sampled on a timer; kernels run
// undisturbed and concurrently, unlike ncu, which serialises kernels and so
// cannot profile collectives whose kernels wait on each other).  NVML's
// NVLink throughput fields and `nvidia-smi nvlink -gt d` report N/A on the
// pool's driver (profiles/r02/nvsmi.txt), so bench.py reads the link counters
// here: nvlrx__bytes / nvltx__bytes (32 B granularity, all links) and their
// user-data parts.
//
// Measurement tooling, not part of the FTAR data plane.  Build:
//   g++ -O2 -shared -fPIC -I$CUDA/include tools/nvlink_pm.cpp -L$CUDA/lib64 -lcupti -o tools/_build/libnvlink_pm.so
#include <cupti_pmsampling.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_target.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

// default metric set; nvpm_open takes any comma-separated list of up to 8
const char* kDefault = "nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum";
constexpr int kMaxMetrics = 8;

struct Sampler {
  bool open = false;
  int device = -1;
  CUpti_Profiler_Host_Object* host = nullptr;
  CUpti_PmSampling_Object* pm = nullptr;
  std::vector<uint8_t> config, counter_data;
  std::vector<std::string> names;
  std::vector<const char*> metrics;
};
Sampler g_s[16];

bool ok(CUptiResult r, const char* what) {
  if (r == CUPTI_SUCCESS) return true;
  const char* s = nullptr;
  cuptiGetResultString(r, &s);
  g_err = std::string(what) + ": " + (s ? s : "?");
  return false;
}

bool reset_counter_data(Sampler& S) {
  CUpti_PmSampling_CounterDataImage_Initialize_Params p{CUpti_PmSampling_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  p.pPmSamplingObject = S.pm;
  p.counterDataSize = S.counter_data.size();
  p.pCounterData = S.counter_data.data();
  return ok(cuptiPmSamplingCounterDataImageInitialize(&p), "cuptiPmSamplingCounterDataImageInitialize");
}

}  // namespace

extern "C" {

const char* nvpm_error(void) { return g_err.c_str(); }

// Prepare PM sampling of `device` every `interval_ns` (at most `max_samples`
// samples per window).  Returns 0 on success.
int nvpm_open(int device, uint64_t interval_ns, uint32_t max_samples, const char* metrics_csv) {
  if (device < 0 || device >= 16) return (g_err = "bad device", 1);
  Sampler& S = g_s[device];
  if (S.open) return 0;
  {
    std::string all = (metrics_csv && *metrics_csv) ? metrics_csv : kDefault;
    size_t pos = 0;
    while (pos <= all.size() && (int)S.names.size() < kMaxMetrics) {
      const size_t q = all.find(',', pos);
      S.names.push_back(all.substr(pos, q == std::string::npos ? std::string::npos : q - pos));
      if (q == std::string::npos) break;
      pos = q + 1;
    }
    for (auto& n : S.names) S.metrics.push_back(n.c_str());
  }
  const char** kMetrics = S.metrics.data();
  const size_t kNumMetrics = S.metrics.size();
  CUpti_Profiler_Initialize_Params pi{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
  if (!ok(cuptiProfilerInitialize(&pi), "cuptiProfilerInitialize")) return 1;
  CUpti_Device_GetChipName_Params cn{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
  cn.deviceIndex = (size_t)device;
  if (!ok(cuptiDeviceGetChipName(&cn), "cuptiDeviceGetChipName")) return 1;
  CUpti_PmSampling_GetCounterAvailability_Params ca{CUpti_PmSampling_GetCounterAvailability_Params_STRUCT_SIZE};
  ca.deviceIndex = (size_t)device;
  if (!ok(cuptiPmSamplingGetCounterAvailability(&ca), "cuptiPmSamplingGetCounterAvailability")) return 1;
  std::vector<uint8_t> avail(ca.counterAvailabilityImageSize);
  ca.pCounterAvailabilityImage = avail.data();
  if (!ok(cuptiPmSamplingGetCounterAvailability(&ca), "cuptiPmSamplingGetCounterAvailability")) return 1;

  CUpti_Profiler_Host_Initialize_Params hi{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
  hi.profilerType = CUPTI_PROFILER_TYPE_PM_SAMPLING;
  hi.pChipName = cn.pChipName;
  hi.pCounterAvailabilityImage = avail.data();
  if (!ok(cuptiProfilerHostInitialize(&hi), "cuptiProfilerHostInitialize")) return 1;
  S.host = hi.pHostObject;
  CUpti_Profiler_Host_ConfigAddMetrics_Params am{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
  am.pHostObject = S.host;
  am.ppMetricNames = kMetrics;
  am.numMetrics = kNumMetrics;
  if (!ok(cuptiProfilerHostConfigAddMetrics(&am), "cuptiProfilerHostConfigAddMetrics")) return 1;
  CUpti_Profiler_Host_GetConfigImageSize_Params cs{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
  cs.pHostObject = S.host;
  if (!ok(cuptiProfilerHostGetConfigImageSize(&cs), "cuptiProfilerHostGetConfigImageSize")) return 1;
  S.config.resize(cs.configImageSize);
  CUpti_Profiler_Host_GetConfigImage_Params gc{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
  gc.pHostObject = S.host;
  gc.pConfigImage = S.config.data();
  gc.configImageSize = S.config.size();
  if (!ok(cuptiProfilerHostGetConfigImage(&gc), "cuptiProfilerHostGetConfigImage")) return 1;

  CUpti_PmSampling_Enable_Params en{CUpti_PmSampling_Enable_Params_STRUCT_SIZE};
  en.deviceIndex = (size_t)device;
  if (!ok(cuptiPmSamplingEnable(&en), "cuptiPmSamplingEnable")) return 1;
  S.pm = en.pPmSamplingObject;
  CUpti_PmSampling_SetConfig_Params sc{CUpti_PmSampling_SetConfig_Params_STRUCT_SIZE};
  sc.pPmSamplingObject = S.pm;
  sc.configSize = S.config.size();
  sc.pConfig = S.config.data();
  sc.hardwareBufferSize = 256ull << 20;
  sc.samplingInterval = interval_ns;
  sc.triggerMode = CUPTI_PM_SAMPLING_TRIGGER_MODE_GPU_TIME_INTERVAL;
  sc.hwBufferAppendMode = CUPTI_PM_SAMPLING_HARDWARE_BUFFER_APPEND_MODE_KEEP_OLDEST;
  if (!ok(cuptiPmSamplingSetConfig(&sc), "cuptiPmSamplingSetConfig")) return 1;
  CUpti_PmSampling_GetCounterDataSize_Params ds{CUpti_PmSampling_GetCounterDataSize_Params_STRUCT_SIZE};
  ds.pPmSamplingObject = S.pm;
  ds.pMetricNames = kMetrics;
  ds.numMetrics = kNumMetrics;
  ds.maxSamples = max_samples;
  if (!ok(cuptiPmSamplingGetCounterDataSize(&ds), "cuptiPmSamplingGetCounterDataSize")) return 1;
  S.counter_data.resize(ds.counterDataSize);
  if (!reset_counter_data(S)) return 1;
  S.open = true;
  S.device = device;
  return 0;
}

int nvpm_start(int device) {
  Sampler& S = g_s[device];
  if (!S.open) return (g_err = "not open", 1);
  if (!reset_counter_data(S)) return 1;
  CUpti_PmSampling_Start_Params st{CUpti_PmSampling_Start_Params_STRUCT_SIZE};
  st.pPmSamplingObject = S.pm;
  return ok(cuptiPmSamplingStart(&st), "cuptiPmSamplingStart") ? 0 : 1;
}

// Stop and sum the window's samples: out[k] = metric k over the window (in
// the order given to nvpm_open); *samples = completed samples; *span_ns =
// first sample start to last sample end.
int nvpm_stop(int device, double* out, int* samples, uint64_t* span_ns, int* overflow) {
  Sampler& S = g_s[device];
  if (!S.open) return (g_err = "not open", 1);
  const char** kMetrics = S.metrics.data();
  const size_t kNumMetrics = S.metrics.size();
  CUpti_PmSampling_Stop_Params sp{CUpti_PmSampling_Stop_Params_STRUCT_SIZE};
  sp.pPmSamplingObject = S.pm;
  if (!ok(cuptiPmSamplingStop(&sp), "cuptiPmSamplingStop")) return 1;
  int ovf = 0;
  for (int guard = 0; guard < 64; ++guard) {
    CUpti_PmSampling_DecodeData_Params dd{CUpti_PmSampling_DecodeData_Params_STRUCT_SIZE};
    dd.pPmSamplingObject = S.pm;
    dd.pCounterDataImage = S.counter_data.data();
    dd.counterDataImageSize = S.counter_data.size();
    if (!ok(cuptiPmSamplingDecodeData(&dd), "cuptiPmSamplingDecodeData")) return 1;
    ovf |= dd.overflow;
    if (dd.decodeStopReason != CUPTI_PM_SAMPLING_DECODE_STOP_REASON_OTHER) break;
  }
  CUpti_PmSampling_GetCounterDataInfo_Params gi{CUpti_PmSampling_GetCounterDataInfo_Params_STRUCT_SIZE};
  gi.pCounterDataImage = S.counter_data.data();
  gi.counterDataImageSize = S.counter_data.size();
  if (!ok(cuptiPmSamplingGetCounterDataInfo(&gi), "cuptiPmSamplingGetCounterDataInfo")) return 1;
  double sum[kMaxMetrics] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t t_first = 0, t_last = 0;
  for (size_t i = 0; i < gi.numCompletedSamples; ++i) {
    CUpti_PmSampling_CounterData_GetSampleInfo_Params si{CUpti_PmSampling_CounterData_GetSampleInfo_Params_STRUCT_SIZE};
    si.pPmSamplingObject = S.pm;
    si.pCounterDataImage = S.counter_data.data();
    si.counterDataImageSize = S.counter_data.size();
    si.sampleIndex = i;
    if (!ok(cuptiPmSamplingCounterDataGetSampleInfo(&si), "cuptiPmSamplingCounterDataGetSampleInfo")) return 1;
    if (i == 0) t_first = si.startTimestamp;
    t_last = si.endTimestamp;
    double v[kMaxMetrics];
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = S.host;
    ev.pCounterDataImage = S.counter_data.data();
    ev.counterDataImageSize = S.counter_data.size();
    ev.ppMetricNames = kMetrics;
    ev.numMetrics = kNumMetrics;
    ev.rangeIndex = i;
    ev.pMetricValues = v;
    if (!ok(cuptiProfilerHostEvaluateToGpuValues(&ev), "cuptiProfilerHostEvaluateToGpuValues")) return 1;
    for (size_t k = 0; k < kNumMetrics; ++k) sum[k] += v[k];
  }
  for (size_t k = 0; k < kNumMetrics; ++k) out[k] = sum[k];
  if (samples) *samples = (int)gi.numCompletedSamples;
  if (span_ns) *span_ns = t_last - t_first;
  if (overflow) *overflow = ovf;
  return 0;
}

int nvpm_close(int device) {
  Sampler& S = g_s[device];
  if (!S.open) return 0;
  CUpti_PmSampling_Disable_Params di{CUpti_PmSampling_Disable_Params_STRUCT_SIZE};
  di.pPmSamplingObject = S.pm;
  cuptiPmSamplingDisable(&di);
  CUpti_Profiler_Host_Deinitialize_Params hd{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
  hd.pHostObject = S.host;
  cuptiProfilerHostDeinitialize(&hd);
  S = Sampler{};
  return 0;
}

}  // extern "C"
