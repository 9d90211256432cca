#include <cuda_runtime.h>
__global__ void k(float* out, const float* __restrict__ xs, const float2* __restrict__ ws, int n) {
  float2 acc0 = make_float2(0,0), acc1 = make_float2(0,0);
  for (int i = 0; i < n; i++) {
    float x = xs[i * 32 + threadIdx.x];
    float2 w0 = ws[i], w1 = ws[i + n];
    acc0 = __ffma2_rn(make_float2(x, x), w0, acc0);
    acc1 = __ffma2_rn(w1, make_float2(x, x), acc1);
  }
  out[threadIdx.x] = acc0.x + acc0.y + acc1.x + acc1.y;
}
