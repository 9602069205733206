// Microbenchmarks on the B200: FP64 FMA latency/throughput, LDS/SHFL latency, barrier cost.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, int n) {
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int ILP>
__global__ void thr_dfma(double* out, long long* cyc, int n) {
  double a[ILP];
  for (int k = 0; k < ILP; ++k) a[k] = out[threadIdx.x] + k;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < ILP; ++k) a[k] = fma(a[k], b, c);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < ILP; ++k) s += a[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) % 1024;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double* out, long long* cyc, int n) {
  double v = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_bar(double* out, long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_div(double* out, long long* cyc, int n) {
  double a = out[threadIdx.x] + 3.0, b = 1.7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = b / a + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_sqrt(double* out, long long* cyc, int n) {
  double a = out[threadIdx.x] + 3.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  cudaMalloc(&c, 64);
  long long h;
  const int n = 4096;
  auto run = [&](const char* name, auto kern, int threads, double ops_per_thread) {
    kern<<<1, threads>>>(d, c, n);
    kern<<<1, threads>>>(d, c, n);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s threads %5d: %8.2f cycles/iter  (%.2f warp-ops/cycle/SM)\n", name, threads, double(h) / n,
           ops_per_thread * threads / 32.0 * n / double(h));
  };
  run("dfma latency", lat_dfma, 32, 1);
  run("dfma thr ilp4", thr_dfma<4>, 128, 4);
  run("dfma thr ilp4", thr_dfma<4>, 512, 4);
  run("dfma thr ilp8", thr_dfma<8>, 1024, 8);
  run("lds latency (dep chain)", lat_lds, 32, 1);
  run("shfl.f64 latency", lat_shfl, 32, 1);
  run("div.f64 latency", lat_div, 32, 1);
  run("sqrt.f64 latency", lat_sqrt, 32, 1);
  run("syncthreads 128", lat_bar, 128, 1);
  run("syncthreads 512", lat_bar, 512, 1);
  run("syncthreads 1024", lat_bar, 1024, 1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
