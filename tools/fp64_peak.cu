// Microbenchmark: FP64 throughput of DFMA vs DMMA (mma.sync f64 shapes) on sm_100a.
// Decides the instruction path of the fp64 A-pass kernels.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

template <int SHAPE>
__global__ void k_dmma(double* out, int iters) {
  // SHAPE 0: m8n8k4, 1: m16n8k4, 2: m16n8k8, 3: m16n8k16
  double acc[4][4];
  for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a[j]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3]) : "d"(a[j]), "d"(a[j+1]), "d"(b[0]));
      } else if (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                     : "d"(a[j]), "d"(a[j+1]), "d"(a[j+2]), "d"(a[j+3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  int sms = p.multiProcessorCount;
  for (int occ : {1, 2, 4, 8}) {
    int blocks = sms * occ, threads = 256, iters = 2000;
    float ms = run(k_dfma, blocks, threads, iters, d);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("DFMA occ %d: %.3f ms  %.2f TFLOP/s\n", occ, ms, flops / ms / 1e9);
  }
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const int mnk[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int s = 0; s < 4; ++s) {
    for (int occ : {1, 2, 4}) {
      int blocks = sms * occ, threads = 256, iters = 1000;
      float ms;
      if (s == 0) ms = run(k_dmma<0>, blocks, threads, iters, d);
      else if (s == 1) ms = run(k_dmma<1>, blocks, threads, iters, d);
      else if (s == 2) ms = run(k_dmma<2>, blocks, threads, iters, d);
      else ms = run(k_dmma<3>, blocks, threads, iters, d);
      double flops = 2.0 * mnk[s] * (blocks * threads / 32.0) * iters * 4;
      printf("DMMA %s occ %d: %.3f ms  %.2f TFLOP/s\n", names[s], occ, ms, flops / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
