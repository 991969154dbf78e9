// probe.cu — microbenchmark of the SFU exp2 rate, the denominator of the exact-KDE
// kernel's MUFU roofline (bench.py `roofline.sfu`).  Every thread runs 8 independent
// ex2.approx.ftz.f32 chains (enough ILP to keep the XU pipe busy), one persistent
// wave of CTAs per SM; ex2/s = total ex2 / kernel time (CUDA events).
#include "internal.h"
#include "ptx.cuh"

namespace dk {
namespace {

__global__ void __launch_bounds__(256) ex2_probe_kernel(int32_t iters, float seed, float* __restrict__ sink) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed * float(threadIdx.x + i) * 1e-9f - 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ex2_approx(v[i]) - 1.5f;  // stays in (-1.5, -0.5]: no denormals
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) sink[threadIdx.x] = s;  // never true; keeps the chains alive
}

}  // namespace
}  // namespace dk

using namespace dk;

extern "C" {

dk_status dk_mufu_probe(int32_t device, double* ex2_per_second) {
  DK_NVTX();
  return guard([&] {
    DK_REQUIRE(ex2_per_second != nullptr, "NULL argument");
    DeviceGuard g(device);
    int sms = 0;
    DK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    float* sink = nullptr;
    DK_CUDA(cudaMalloc(&sink, 256 * sizeof(float)));
    cudaEvent_t e0, e1;
    DK_CUDA(cudaEventCreate(&e0));
    DK_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8, iters = 4096;  // 8 CTAs x 256 threads = 64 warps per SM
    ex2_probe_kernel<<<blocks, 256>>>(64, 1.f, sink);  // warm-up
    DK_CHECK_LAUNCH();
    DK_CUDA(cudaEventRecord(e0));
    ex2_probe_kernel<<<blocks, 256>>>(iters, 1.f, sink);
    DK_CHECK_LAUNCH();
    DK_CUDA(cudaEventRecord(e1));
    DK_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    DK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    *ex2_per_second = double(blocks) * 256.0 * iters * 8.0 / (double(ms) * 1e-3);
  });
}

}  // extern "C"
