// energy.cu — NVML energy measurement for the objective-aware tuner (the
// paper's four objectives: latency, energy, average power and MFLOPS/W,
// P:66). libnvidia-ml is loaded lazily (dlopen), so the library
// has no link-time NVML dependency. Energy = delta of the device's total
// energy counter over a window of back-to-back SpMVs (reading R18: counter
// delta over a busy window instead of the paper's power sampling thread).
#include <dlfcn.h>

#include <mutex>

#include "spmv_common.cuh"

namespace spmv {
namespace {

struct NvmlApi {
  void* lib = nullptr;
  int (*Init)() = nullptr;
  int (*HandleByPci)(const char*, void**) = nullptr;
  int (*TotalEnergy)(void*, unsigned long long*) = nullptr;
};

NvmlApi* nvml_api() {
  static NvmlApi api;
  static bool ok = false;
  static std::once_flag once;
  std::call_once(once, [] {
    void* l = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!l) l = dlopen("libnvidia-ml.so", RTLD_NOW | RTLD_LOCAL);
    if (!l) return;
    api.lib = l;
    api.Init = (decltype(api.Init))dlsym(l, "nvmlInit_v2");
    api.HandleByPci = (decltype(api.HandleByPci))dlsym(l, "nvmlDeviceGetHandleByPciBusId_v2");
    api.TotalEnergy = (decltype(api.TotalEnergy))dlsym(l, "nvmlDeviceGetTotalEnergyConsumption");
    ok = api.Init && api.HandleByPci && api.TotalEnergy && api.Init() == 0;
  });
  return ok ? &api : nullptr;
}

void* nvml_device(int device) {
  NvmlApi* api = nvml_api();
  if (!api) fail(SPMV_ERR_NVML, "libnvidia-ml not available (energy objectives need NVML)");
  char bus[32];
  CK(cudaDeviceGetPCIBusId(bus, (int)sizeof(bus), device));
  void* dev = nullptr;
  if (api->HandleByPci(bus, &dev) != 0 || !dev) fail(SPMV_ERR_NVML, std::string("NVML has no device ") + bus);
  return dev;
}

}  // namespace

// Run `launch` back-to-back for at least min_seconds (device time) and
// return the window's time (CUDA events) and energy (NVML counter delta).
EnergySample measure_energy(spmv_matrix* h, const std::function<void()>& launch, double min_seconds) {
  void* dev = nvml_device(h->device);
  NvmlApi* api = nvml_api();
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaStreamSynchronize(h->stream));
  unsigned long long e0 = 0, e1 = 0;
  api->TotalEnergy(dev, &e0);
  CK(cudaEventRecord(a, h->stream));
  int64_t reps = 0;
  int64_t batch = 8;
  float ms = 0.f;
  while (true) {
    for (int64_t i = 0; i < batch; ++i) launch();
    reps += batch;
    CK(cudaEventRecord(b, h->stream));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms * 1e-3 >= min_seconds) break;
    const double per = ms / (double)reps;
    const double need = (min_seconds * 1e3 - ms) / (per > 1e-6 ? per : 1e-6);
    batch = (int64_t)(need > 1 ? need : 1);
    if (batch > 100000) batch = 100000;
  }
  api->TotalEnergy(dev, &e1);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  EnergySample s;
  s.seconds = ms * 1e-3;
  s.joules = (double)(e1 - e0) * 1e-3;
  s.reps = reps;
  s.watts = s.seconds > 0 ? s.joules / s.seconds : 0.0;
  return s;
}

bool nvml_available() { return nvml_api() != nullptr; }

}  // namespace spmv
