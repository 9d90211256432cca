// Shared-memory LDS.32 throughput for the access patterns of the transform's
// window loads (consecutive / misaligned / stride-7 lanes).
#include <cstdio>
#include <cuda_runtime.h>

template <int STRIDE, int OFFSET>
__global__ void lds(float* out, int iters, int step) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int base = (threadIdx.x >> 5) * 64 + OFFSET + lane * STRIDE;
  float acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int q = 0; q < 16; q++) acc += s[(base + q * step) & 8191];
    base = (base + 32 * 16) & 4095;
  }
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

template <int STRIDE, int OFFSET>
void run(const char* name, float* out, int sms, int step) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, tpb = 512, grid = sms * 2;
  lds<STRIDE, OFFSET><<<grid, tpb>>>(out, iters, step);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    lds<STRIDE, OFFSET><<<grid, tpb>>>(out, iters, step);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double lds_per_sm = (double)grid * (tpb / 32) * iters * 16 / sms;
  double cycles = best * 1e-3 * 1.965e9;
  printf("{\"pattern\": \"%s\", \"step\": %d, \"cycles_per_warp_lds_per_sm\": %.3f}\n", name, step, cycles / lds_per_sm);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 16);
  for (int step : {32, 7, 100}) {
    run<1, 0>("consecutive_aligned", out, sms, step);
    run<1, 1>("consecutive_off1", out, sms, step);
    run<1, 16>("consecutive_off16", out, sms, step);
    run<7, 0>("stride7", out, sms, step);
    run<7, 3>("stride7_off3", out, sms, step);
    run<2, 0>("stride2_2way", out, sms, step);
  }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
