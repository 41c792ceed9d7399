// Latency calibration on sm_100a: dependent DFMA chain, dependent LDS
// (pointer chase in shared memory), generic-pointer load chain into shared
// memory, __syncthreads round trip at 384 threads, fast FP64 reciprocal.
#include <cstdio>

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  r = r * fma(-x, r, 2.0);
  return r;
}

__global__ void __launch_bounds__(384, 1) probe(long long* cyc, double* sink, int* isink, int N) {
  __shared__ int chase[1024];
  __shared__ double dch[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { chase[i] = (i * 37 + 11) & 1023; dch[i] = 1.0 + 1e-9 * i; }
  __syncthreads();
  double x = 1.0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 1.0000001, 1e-12);
  long long t1 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < N; ++i) p = chase[p];
  long long t2 = clock64();
  // generic pointer chase (compiler cannot prove shared space)
  volatile int* gp = (volatile int*)((threadIdx.x < 1000) ? (int*)chase : (int*)isink);
  int q = threadIdx.x & 1023;
  for (int i = 0; i < N; ++i) q = gp[q];
  long long t3 = clock64();
  for (int i = 0; i < N; ++i) __syncthreads();
  long long t4 = clock64();
  double y = 3.0 + threadIdx.x;
  for (int i = 0; i < N; ++i) y = fast_rcp(y) + 2.0;
  long long t5 = clock64();
  double z = 0.0;
  for (int i = 0; i < N; ++i) z = dch[((int)z + i) & 1023] + z * 1e-30;
  long long t6 = clock64();
  double d0 = 0.0, d1 = 0.0, aa = 1.0 + 1e-9 * threadIdx.x, bbv = 0.999;
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(aa), "d"(bbv));
  long long t7 = clock64();
  double e0 = 0, e1 = 0, f0 = 0, f1 = 0, g0 = 0, g1 = 0, h0 = 0, h1 = 0;
  for (int i = 0; i < N; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(aa), "d"(bbv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(aa), "d"(bbv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(g0), "+d"(g1) : "d"(aa), "d"(bbv));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(h0), "+d"(h1) : "d"(aa), "d"(bbv));
  }
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[6] = (t7 - t6) / N; cyc[7] = (t8 - t7) / N;
    cyc[0] = (t1 - t0) / N; cyc[1] = (t2 - t1) / N; cyc[2] = (t3 - t2) / N; cyc[3] = (t4 - t3) / N;
    cyc[4] = (t5 - t4) / N; cyc[5] = (t6 - t5) / N;
  }
  sink[threadIdx.x] = x + y + z + d0 + d1 + e0 + f0 + g0 + h0 + e1 + f1 + g1 + h1;
  isink[threadIdx.x] = p + q;
}

int main() {
  long long* cyc; double* sink; int* isink;
  cudaMalloc(&cyc, 128); cudaMalloc(&sink, 384 * 8); cudaMalloc(&isink, 1024 * 4);
  cudaMemset(isink, 0, 4096);
  probe<<<1, 384>>>(cyc, sink, isink, 2000);
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  printf("cycles per op: DFMA chain %lld | LDS chase %lld | generic-ptr LD chase (smem) %lld | __syncthreads(384) %lld | fast_rcp f64 + add %lld | LDS f64 + DFMA chain %lld | DMMA884 chain %lld | 4 indep DMMA chains %lld per 4 [%s]\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
