#include <cstdio>
#include <cuda_runtime.h>
// issue-bound mixes: 8 FP32 FMAs + K integer ALU ops per iteration, as 8 FFMA or 4 FFMA2
template <int K>
__global__ void k_a(float* out, unsigned* uo, int iters) {
  float x[8]; unsigned u[8];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x * 0.001f + i; u[i] = threadIdx.x * 7 + i; }
  float c = out[1024], d = out[1025]; unsigned m = uo[0];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], c, d);
#pragma unroll
    for (int i = 0; i < K; i++) u[i] = (u[i] ^ m) ^ (u[i] >> 3);
  }
  float s = 0; unsigned t = 0; for (int i = 0; i < 8; i++) { s += x[i]; t += u[i]; }
  if (s == 12345.f || t == 77u) out[threadIdx.x] = s + t;
}
template <int K>
__global__ void k_b(float* out, unsigned* uo, int iters) {
  float2 x[4]; unsigned u[8];
  for (int i = 0; i < 4; i++) x[i] = make_float2(threadIdx.x * 0.001f + i, i);
  for (int i = 0; i < 8; i++) u[i] = threadIdx.x * 7 + i;
  float2 c = make_float2(out[1024], out[1026]), d = make_float2(out[1025], out[1027]); unsigned m = uo[0];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) x[i] = __ffma2_rn(x[i], c, d);
#pragma unroll
    for (int i = 0; i < K; i++) u[i] = (u[i] ^ m) ^ (u[i] >> 3);
  }
  float s = 0; unsigned t = 0; for (int i = 0; i < 4; i++) s += x[i].x + x[i].y; for (int i = 0; i < 8; i++) t += u[i];
  if (s == 12345.f || t == 77u) out[threadIdx.x] = s + t;
}
int main() {
  float* d; unsigned* u;
  cudaMalloc(&d, 8192 * 4); cudaMemset(d, 0, 8192 * 4);
  cudaMalloc(&u, 64); cudaMemset(u, 0, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000, blocks = sms * 8, thr = 256;
  auto run = [&](const char* name, auto fn) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 3; r++) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    double cyc = ms * 1e-3 * 1.965e9 / ((double)blocks * thr / 32 / (sms * 4)) / iters;  // SMSP cycles per warp-iteration
    printf("%-14s %8.3f ms  %6.2f SMSP cycles per warp iteration  %s\n", name, ms, cyc, cudaGetErrorString(cudaGetLastError()));
  };
  run("8ffma+0int", [&] { k_a<0><<<blocks, thr>>>(d, u, iters); });
  run("4ffma2+0int", [&] { k_b<0><<<blocks, thr>>>(d, u, iters); });
  run("8ffma+4int", [&] { k_a<4><<<blocks, thr>>>(d, u, iters); });
  run("4ffma2+4int", [&] { k_b<4><<<blocks, thr>>>(d, u, iters); });
  run("8ffma+8int", [&] { k_a<8><<<blocks, thr>>>(d, u, iters); });
  run("4ffma2+8int", [&] { k_b<8><<<blocks, thr>>>(d, u, iters); });
  return 0;
}
