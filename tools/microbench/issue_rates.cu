#include <cstdio>
#include <cuda_runtime.h>
// issue-rate microbenchmarks: 8 independent chains per thread
template <int K>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  float c = out[1024], d = out[1025];   // runtime registers: 3-reg form
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaf(x[i], c, d);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters) {
  float2 x[8];
  for (int i = 0; i < 8; i++) x[i] = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
  float2 c = make_float2(out[1024], out[1026]), d = make_float2(out[1025], out[1027]);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __ffma2_rn(x[i], c, d);
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i].x + x[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_mix(float* out, unsigned* uo, int iters) {
  // FFMA 3-reg interleaved with LOP3/IADD3 integer ops (alu pipe)
  float x[4]; unsigned u[4];
  for (int i = 0; i < 4; i++) { x[i] = threadIdx.x * 0.001f + i; u[i] = threadIdx.x * 7 + i; }
  float c = out[1024], d = out[1025]; unsigned m = uo[0], n = uo[1];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) { x[i] = fmaf(x[i], c, d); u[i] = (u[i] ^ m) + n; }
  }
  float s = 0; unsigned t = 0; for (int i = 0; i < 4; i++) { s += x[i]; t += u[i]; }
  if (s == 12345.f || t == 77u) out[threadIdx.x] = s + t;
}
__global__ void k_mix2(float* out, unsigned* uo, int iters) {
  float2 x[4]; unsigned u[4];
  for (int i = 0; i < 4; i++) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); u[i] = threadIdx.x * 7 + i; }
  float2 c = make_float2(out[1024], out[1026]), d = make_float2(out[1025], out[1027]); unsigned m = uo[0], n = uo[1];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) { x[i] = __ffma2_rn(x[i], c, d); u[i] = (u[i] ^ m) + n; }
  }
  float s = 0; unsigned t = 0; for (int i = 0; i < 4; i++) { s += x[i].x + x[i].y; t += u[i]; }
  if (s == 12345.f || t == 77u) out[threadIdx.x] = s + t;
}
__global__ void k_fmul(float* out, int iters) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  float c = out[1024];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = x[i] * c;
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_fadd_fmul(float* out, int iters) {
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  float c = out[1024];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i+=2) { x[i] = x[i] * c; x[i+1] = x[i+1] + c; }
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void k_sel(float* out, int iters) {
  // FSEL / FMNMX style (alu)
  float x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 0.001f + i;
  float c = out[1024];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fmaxf(x[i], c) ;
    c = c + 1e-7f;
  }
  float s = 0; for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}
int main() {
  float* d; unsigned* u;
  cudaMalloc(&d, 8192 * 4); cudaMemset(d, 0, 8192 * 4);
  cudaMalloc(&u, 64); cudaMemset(u, 0, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000, blocks = sms * 8, thr = 256;
  double thr_total = (double)blocks * thr;
  auto run = [&](const char* name, auto fn, double ops_per_iter) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 3; r++) fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
    double lane_ops = thr_total * iters * ops_per_iter;
    printf("%-12s %8.3f ms  %7.2f T lane-ops/s  (%5.3f per SM per clk @%d MHz)  err=%s\n", name, ms,
           lane_ops / ms / 1e9, lane_ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("ffma", [&] { k_ffma<0><<<blocks, thr>>>(d, 1.f, 2.f, iters); }, 8);
  run("ffma2(x2)", [&] { k_ffma2<<<blocks, thr>>>(d, iters); }, 16);
  run("mix f+i", [&] { k_mix<<<blocks, thr>>>(d, u, iters); }, 8);
  run("mix2 f2+i", [&] { k_mix2<<<blocks, thr>>>(d, u, iters); }, 12);
  run("fmul", [&] { k_fmul<<<blocks, thr>>>(d, iters); }, 8);
  run("fadd/fmul", [&] { k_fadd_fmul<<<blocks, thr>>>(d, iters); }, 8);
  run("fmnmx", [&] { k_sel<<<blocks, thr>>>(d, iters); }, 8);
  return 0;
}
