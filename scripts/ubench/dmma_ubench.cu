// Microbenchmark: FP64 tensor-core MMA throughput on sm_100a, mma.sync m8n8k4 vs m16n8k4/k8/k16.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1684(double (&d)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void dmma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int MODE, int ILP>
__global__ void k(double* out, int n) {
  double acc[ILP][4];
  for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = threadIdx.x * 1e-3 + i + j;
  double a[8], b[4];
  for (int j = 0; j < 8; ++j) a[j] = 1.0 + 1e-9 * (threadIdx.x + j);
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - 1e-9 * (threadIdx.x + j);
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (MODE == 0) { dmma884(acc[i][0], acc[i][1], a[0], b[0]); dmma884(acc[i][2], acc[i][3], a[1], b[1]); }
      if (MODE == 1) { double aa[2] = {a[0], a[1]}; dmma1684(acc[i], aa, b[0]); }
      if (MODE == 2) { double aa[4] = {a[0], a[1], a[2], a[3]}; double bb[2] = {b[0], b[1]}; dmma1688(acc[i], aa, bb); }
      if (MODE == 3) { dmma16816(acc[i], a, b); }
    }
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int ILP>
void run(const char* name, double flops_per_warp_iter, int threads) {
  double* d;
  cudaMalloc(&d, 148 * 4 * 1024 * 8);
  const int n = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE, ILP><<<148 * 2, threads>>>(d, 100);
  cudaEventRecord(e0);
  k<MODE, ILP><<<148 * 2, threads>>>(d, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = flops_per_warp_iter * ILP * double(n) * (threads / 32) * 148 * 2;
  printf("%-14s ilp %d threads %4d x2 CTAs/SM: %8.3f ms  %7.2f TFLOP/s  (%s)\n", name, ILP, threads, ms, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<0, 4>("m8n8k4 x2", 2 * 2.0 * 8 * 8 * 4, 256);
  run<0, 8>("m8n8k4 x2", 2 * 2.0 * 8 * 8 * 4, 512);
  run<1, 4>("m16n8k4", 2.0 * 16 * 8 * 4, 256);
  run<1, 8>("m16n8k4", 2.0 * 16 * 8 * 4, 512);
  run<2, 4>("m16n8k8", 2.0 * 16 * 8 * 8, 256);
  run<2, 8>("m16n8k8", 2.0 * 16 * 8 * 8, 512);
  run<3, 4>("m16n8k16", 2.0 * 16 * 8 * 16, 256);
  run<3, 8>("m16n8k16", 2.0 * 16 * 8 * 16, 512);
  run<3, 2>("m16n8k16", 2.0 * 16 * 8 * 16, 128);
  return 0;
}
