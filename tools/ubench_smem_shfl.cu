// Micro-benchmark: does SHFL share the shared-memory crossbar bandwidth with LDS on sm_100a?
// (DESIGN.md §10 round 2: the high-order sweeps are bound by 128 B/clk/SM of LDS traffic.)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_smem_shfl.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

template <int MODE>   // 0: LDS.64 x4; 1: SHFL.32 x8; 2: LDS.64 x4 + SHFL.32 x8; 3: LDS.128 x2; 4: LDS.32 x8
__global__ void __launch_bounds__(512, 1) kern(float* out, unsigned long long* cyc, int zero) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  float a0 = lane, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
  float b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0, b6 = 0, b7 = 0;
  float s0 = lane, s1 = lane + 1, s2 = lane + 2, s3 = lane + 3, s4 = lane + 4, s5 = lane + 5, s6 = lane + 6, s7 = lane + 7;
  unsigned base = (unsigned)__cvta_generic_to_shared(sm) + (w * 64 + lane * 2) * 4;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITER; ++it) {
    const unsigned off = ((it * 2048) & 16383) + (zero & it);
    if (MODE == 0 || MODE == 2) {
      float x, y;
#define L64(k, A, B)                                                                            \
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(base + off + k * 256)); \
  A += x; B += y;
      L64(0, a0, a1) L64(1, a2, a3) L64(2, a4, a5) L64(3, a6, a7)
    }
    if (MODE == 3) {
      float x, y, z, v;
      unsigned b4 = (unsigned)__cvta_generic_to_shared(sm) + (w * 128 + lane * 4) * 4;
#define L128(k, A, B, C, D)                                                                      \
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(v)     \
               : "r"(b4 + ((off * 2) & 16383) + k * 512));                                      \
  A += x; B += y; C += z; D += v;
      L128(0, a0, a1, a2, a3) L128(1, a4, a5, a6, a7)
    }
    if (MODE == 4) {
      float x;
      unsigned b1 = (unsigned)__cvta_generic_to_shared(sm) + (w * 32 + lane) * 4;
#define L32(k, A)                                                                      \
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(b1 + (off & 8191) + k * 128)); A += x;
      L32(0, a0) L32(1, a1) L32(2, a2) L32(3, a3) L32(4, a4) L32(5, a5) L32(6, a6) L32(7, a7)
    }
    if (MODE == 1 || MODE == 2) {
      b0 += __shfl_sync(0xffffffffu, s0, lane + 1);
      b1 += __shfl_sync(0xffffffffu, s1, lane + 2);
      b2 += __shfl_sync(0xffffffffu, s2, lane + 3);
      b3 += __shfl_sync(0xffffffffu, s3, lane + 5);
      b4 += __shfl_sync(0xffffffffu, s4, lane + 31);
      b5 += __shfl_sync(0xffffffffu, s5, lane + 30);
      b6 += __shfl_sync(0xffffffffu, s6, lane + 29);
      b7 += __shfl_sync(0xffffffffu, s7, lane + 27);
      s0 += 1.f; s1 += 1.f; s2 += 1.f; s3 += 1.f; s4 += 1.f; s5 += 1.f; s6 += 1.f; s7 += 1.f;
    }
  }
  const long long t1 = clock64();
  float r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + b0 + b1 + b2 + b3 + b4 + b5 + b6 + b7;
  if (r == 1234.5f) out[threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE>
void run(const char* name, int nthreads, int nsm, float* out, unsigned long long* cyc) {
  kern<MODE><<<nsm, nthreads>>>(out, cyc, 0);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<nsm, nthreads>>>(out, cyc, 0);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double c = 0; for (int i = 0; i < nsm; ++i) c += h[i]; c /= nsm;
  const double warps = nthreads / 32.0, per = c / ITER;   // cycles per iteration per SM
  double lds_b = 0, shfl = 0;
  if (MODE == 0 || MODE == 2) lds_b = warps * 4 * 256;
  if (MODE == 3) lds_b = warps * 2 * 512;
  if (MODE == 4) lds_b = warps * 8 * 128;
  if (MODE == 1 || MODE == 2) shfl = warps * 8;
  printf("%-22s thr %4d  cyc/iter %8.2f  LDS B/clk/SM %7.2f  SHFL warp-instr/clk/SM %6.3f  (%.3f ms, %s)\n",
         name, nthreads, per, lds_b / per, shfl / per, ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 1024 * 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 512}) {
    run<0>("LDS.64 x4", t, nsm, out, cyc);
    run<3>("LDS.128 x2", t, nsm, out, cyc);
    run<4>("LDS.32 x8", t, nsm, out, cyc);
    run<1>("SHFL.32 x8", t, nsm, out, cyc);
    run<2>("LDS.64 x4 + SHFL x8", t, nsm, out, cyc);
  }
  return 0;
}
