// FP32 pipe microbenchmark: measures the B200 FP32 roofline denominator
// (FFMA / FFMA2 / FMUL+FADD issue rates) with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

#define NACC 16
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
// conv-like: w shared across positions (reuse), x differs
__global__ void k_ffma_conv(float* out, const float* win, int iters) {
  float acc[NACC], x[NACC + 8], w[9];
#pragma unroll
  for (int i = 0; i < NACC + 8; i++) x[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 9; i++) w[i] = win[i];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int m = 0; m < 9; m++)
#pragma unroll
      for (int r = 0; r < NACC; r++) acc[r] = fmaf(w[m], x[r + (m & 7)], acc[r]);
#pragma unroll
    for (int i = 0; i < 9; i++) w[i] = w[i] * 0.999f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  float2 acc[NACC / 2];
  float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) acc[i] = __ffma2_rn(acc[i], a2, b2);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_mul_add(float* out, float a, float b, int iters) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = __fadd_rn(__fmul_rn(acc[i], a), b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_mul2_add2(float* out, float a, float b, int iters) {
  float2 acc[NACC / 2];
  float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) acc[i] = __fadd2_rn(__fmul2_rn(acc[i], a2), b2);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

// exact packed: FMUL2 then FFMA2 with an opaque 1.0 multiplier (ptxas cannot fuse it)
__global__ void k_mul2_one(float* out, float a, float b, float one, int iters) {
  float2 acc[NACC / 2];
  float2 a2 = make_float2(a, a), b2 = make_float2(b, b), o2 = make_float2(one, one);
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC / 2; i++) acc[i] = __ffma2_rn(__fmul2_rn(acc[i], a2), o2, b2);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC / 2; i++) s += acc[i].x + acc[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, clk);
  float* out; cudaMalloc(&out, 1 << 20);
  float* win; cudaMalloc(&win, 64); cudaMemset(win, 0, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int tpb : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      if (tpb * bps > 2048) continue;
      int grid = p.multiProcessorCount * bps;
      for (int v = 0; v < 6; v++) {
        auto launch = [&]() {
          switch (v) {
            case 0: k_ffma<<<grid, tpb>>>(out, 0.999f, 0.001f, iters); break;
            case 1: k_ffma2<<<grid, tpb>>>(out, 0.999f, 0.001f, iters); break;
            case 2: k_mul_add<<<grid, tpb>>>(out, 0.999f, 0.001f, iters); break;
            case 3: k_mul2_add2<<<grid, tpb>>>(out, 0.999f, 0.001f, iters); break;
            case 4: k_ffma_conv<<<grid, tpb>>>(out, win, iters / 9 * 16 / 16); break;
            case 5: k_mul2_one<<<grid, tpb>>>(out, 0.999f, 0.001f, 1.0f, iters); break;
          }
        };
        launch(); cudaDeviceSynchronize();
        float best = 1e30f;
        for (int rep = 0; rep < 5; rep++) {
          cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        double ops;  // FP32 lane-ops (FMA counted as 2 flops)
        double threads = (double)grid * tpb;
        const char* name;
        switch (v) {
          case 0: name = "ffma"; ops = threads * iters * NACC * 2.0; break;
          case 1: name = "ffma2"; ops = threads * iters * NACC * 2.0; break;
          case 2: name = "fmul_fadd"; ops = threads * iters * NACC * 2.0; break;
          case 3: name = "fmul2_fadd2"; ops = threads * iters * NACC * 2.0; break;
          case 5: name = "fmul2_ffma2one"; ops = threads * iters * NACC * 2.0; break;
          default: name = "ffma_conv"; ops = threads * (iters / 9) * 9.0 * NACC * 2.0; break;
        }
        printf("{\"kernel\": \"%s\", \"tpb\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
               name, tpb, bps, best, ops / best / 1e9);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
