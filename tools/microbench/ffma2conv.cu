// FFMA2 issue-rate microbenchmark for the transform's inner-loop shape:
// acc[p][r] (float2 = one kernel pair) += w[p][j] (float2) * x[r + j] (scalar broadcast).
#include <cstdio>
#include <cuda_runtime.h>

template <int P, int R, int LEN>
__global__ void conv(float* out, const float* __restrict__ win, const float* __restrict__ xin, int iters) {
  float2 w[P][LEN];
  float x[R + LEN - 1];
  float2 acc[P][R];
#pragma unroll
  for (int p = 0; p < P; p++)
#pragma unroll
    for (int j = 0; j < LEN; j++) w[p][j] = make_float2(win[2 * (p * LEN + j)], win[2 * (p * LEN + j) + 1]);
#pragma unroll
  for (int q = 0; q < R + LEN - 1; q++) x[q] = xin[(threadIdx.x + q) & 255];
#pragma unroll
  for (int p = 0; p < P; p++)
#pragma unroll
    for (int r = 0; r < R; r++) acc[p][r] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < LEN; j++)
#pragma unroll
      for (int p = 0; p < P; p++)
#pragma unroll
        for (int r = 0; r < R; r++) acc[p][r] = __ffma2_rn(w[p][j], make_float2(x[r + j], x[r + j]), acc[p][r]);
#pragma unroll
    for (int q = 0; q < R + LEN - 1; q++) x[q] = x[q] * 0.5f + 0.25f;
  }
  float s = 0;
#pragma unroll
  for (int p = 0; p < P; p++)
#pragma unroll
    for (int r = 0; r < R; r++) s += acc[p][r].x + acc[p][r].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int P, int R, int LEN>
void run(const char* name, float* out, float* win, float* xin, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, tpb = 256, grid = sms * 2;
  conv<P, R, LEN><<<grid, tpb>>>(out, win, xin, iters);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    conv<P, R, LEN><<<grid, tpb>>>(out, win, xin, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = (double)grid * tpb * iters * (P * R * LEN * 4.0);  // FFMA2 = 2 FMAs = 4 flops
  printf("{\"kernel\": \"%s\", \"P\": %d, \"R\": %d, \"LEN\": %d, \"tflops\": %.2f, \"fma_only_tflops\": %.2f}\n", name, P, R, LEN,
         flops / best / 1e9, flops / best / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out, *win, *xin;
  cudaMalloc(&out, 4096); cudaMalloc(&win, 4096); cudaMalloc(&xin, 4096);
  cudaMemset(win, 0, 4096); cudaMemset(xin, 0, 4096);
  run<2, 7, 9>("ffma2_conv", out, win, xin, sms);
  run<2, 7, 11>("ffma2_conv", out, win, xin, sms);
  run<2, 5, 9>("ffma2_conv", out, win, xin, sms);
  run<1, 7, 9>("ffma2_conv", out, win, xin, sms);
  run<2, 9, 9>("ffma2_conv", out, win, xin, sms);
  run<4, 4, 9>("ffma2_conv", out, win, xin, sms);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}
