// Latency microbenchmarks on sm_100a: dependent DMMA m8n8k4, DFMA, DP rsqrt,
// shfl, __syncthreads (256 threads), named barrier.  Cycles per op via clock64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int iters) {
  double c0 = threadIdx.x * 1e-3, c1 = 1.0, a = 1.0000001, b = 0.999999;
  long long t0, t1;
  // DMMA chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // independent DMMA x4 (throughput per warp)
  double d0 = c0, d1 = c1, e0 = c0, e1 = c1, f0 = c0, f1 = c1, g0 = c0, g1 = c1;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(g0), "+d"(g1) : "d"(a), "d"(b));
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // DFMA chain
  double x = c0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // rsqrt chain
  double y = 2.0 + c0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = rsqrt(y) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // shfl chain
  double z = c0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // named barrier 224 threads (warps 1..7)
  if (threadIdx.x >= 32) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) asm volatile("bar.sync 1, 224;" ::: "memory");
    t1 = clock64();
    if (threadIdx.x == 32) cyc[6] = (t1 - t0) / iters;
  }
  // smem load-use chain
  __shared__ int sidx[256];
  sidx[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  int p = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = sidx[p];
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / iters;
  // sqrt chain and division chain
  double s = 2.0 + c0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = sqrt(s) + 1.5;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / iters;
  double q = 2.0 + c0;
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) q = 3.0 / q + 1.0;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = (t1 - t0) / iters;
  out[threadIdx.x] = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1 + g0 + g1 + x + y + z + p + s + q;
}

// DMMA throughput per SM: every warp runs 4 independent chains.
__global__ void k_tput(double* out, int iters) {
  double a = 1.0000001, b = 0.999999;
  double r[8];
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(r[2*j]), "+d"(r[2*j+1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma_tput(double* out, int iters) {
  double a = 1.0000001, b = 0.999999;
  double r[8];
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = fma(r[j], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8 * 8); cudaMalloc(&cyc, 64 * 8);
  k_lat<<<1, 256>>>(out, cyc, 1000);
  k_lat<<<1, 256>>>(out, cyc, 1000);
  long long h[16]; cudaMemcpy(h, cyc, 10 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"dmma_dep", "dmma_4indep_per_iter", "dfma_dep", "rsqrt_dep(+dadd)", "shfl_dep(+dadd)",
                         "syncthreads_256", "bar_sync_224", "lds_dep", "sqrt_dep(+dadd)", "ddiv_dep(+dadd)"};
  for (int i = 0; i < 10; ++i) printf("%-24s %lld cycles\n", names[i], h[i]);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {4, 8, 16, 32}) {
    int it = 20000;
    k_tput<<<148, 32 * w>>>(out, 100);
    cudaEventRecord(e0); k_tput<<<148, 32 * w>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * w * it * 4 * 512;  // 8x8x4 FMA = 256 FMA = 512 flop
    printf("DMMA tput warps/SM=%2d: %.2f TFLOP/s\n", w, flops / ms / 1e9);
  }
  for (int w : {8, 16, 32}) {
    int it = 20000;
    k_dfma_tput<<<148, 32 * w>>>(out, 100);
    cudaEventRecord(e0); k_dfma_tput<<<148, 32 * w>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 32 * w * it * 8 * 2;
    printf("DFMA tput warps/SM=%2d: %.2f TFLOP/s\n", w, flops / ms / 1e9);
  }
  return 0;
}
