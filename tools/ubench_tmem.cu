// Micro-benchmark: TMEM -> register bandwidth (tcgen05.ld) on sm_100a, and whether it shares the
// 128 B/clk/SM shared-memory crossbar with LDS (TMEM as z-queue storage).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ut tools/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 2048;

// MODE: 1 = TMEM loads (warps 0..NT-1), 2 = LDS.128 (warps NT..NT+NL-1), 3 = both
template <int MODE, int NT, int NL, int X>
__global__ void __launch_bounds__(32 * (NT + NL), 1) kern(float* out, unsigned long long* cyc, int zero) {
  __shared__ __align__(16) float sm[8192];
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = taddr_s;
  // fill TMEM (every TMEM warp writes its lane quadrant, all 512 columns)
  if (warp < NT && warp < 4) {
    const uint32_t ta = tbase + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < 512; c += 4) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                   :: "r"(ta + c), "r"(lane + c), "r"(lane + c + 1), "r"(lane + c + 2), "r"(lane + c + 3)
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t acc = 0;
  float facc = 0.f;
  const long long t0 = clock64();
  if ((MODE & 1) && warp < NT) {
    const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16);
#pragma unroll 1
    for (int it = 0; it < ITER; ++it) {
      const uint32_t col = ((it * X) & 511) + (zero & it);
      uint32_t r[X];
      if constexpr (X == 16) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(ta + col));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(ta + col));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= r[i];
    }
  }
  if ((MODE & 2) && warp >= NT) {
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + ((warp - NT) * 128 + lane * 4) * 4;
#pragma unroll 4
    for (int it = 0; it < ITER; ++it) {
      const unsigned off = ((it * 2048) & 16383) + (zero & it);
      float x, y, z, w;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
                     : "r"(base + ((off + k * 512) & 16383)));
        facc += x + y + z + w;
      }
    }
  }
  const long long t1 = clock64();
  if (acc == 12345u || facc == 1234.5f) out[threadIdx.x] = facc + acc;
  if (lane == 0) cyc[blockIdx.x * 32 + warp] = (unsigned long long)(t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase) : "memory");
}

template <int MODE, int NT, int NL, int X>
void run(const char* name, int nsm, float* out, unsigned long long* cyc) {
  kern<MODE, NT, NL, X><<<nsm, 32 * (NT + NL)>>>(out, cyc, 0);
  cudaError_t e = cudaDeviceSynchronize();
  kern<MODE, NT, NL, X><<<nsm, 32 * (NT + NL)>>>(out, cyc, 0);
  e = cudaDeviceSynchronize();
  static unsigned long long h[32 * 1024];
  cudaMemcpy(h, cyc, (size_t)nsm * 32 * 8, cudaMemcpyDeviceToHost);
  double ct = 0, cl = 0;
  for (int b = 0; b < nsm; ++b) {
    for (int w = 0; w < NT; ++w) ct = ct > h[b * 32 + w] ? ct : (double)h[b * 32 + w];
    for (int w = NT; w < NT + NL; ++w) cl = cl > h[b * 32 + w] ? cl : (double)h[b * 32 + w];
  }
  const double tb = (MODE & 1) ? (double)NT * ITER * 32 * X * 4 / ct : 0;   // TMEM bytes / clk / SM
  const double lb = (MODE & 2) ? (double)NL * ITER * 4 * 512 / cl : 0;      // LDS bytes / clk / SM
  printf("%-34s TMEM %7.1f B/clk/SM   LDS %7.1f B/clk/SM   (%s)\n", name, tb, lb, cudaGetErrorString(e));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, (size_t)nsm * 32 * 8);
  run<1, 4, 0, 16>("TMEM x16, 4 warps", nsm, out, cyc);
  run<1, 8, 0, 16>("TMEM x16, 8 warps", nsm, out, cyc);
  run<1, 16, 0, 16>("TMEM x16, 16 warps", nsm, out, cyc);
  run<1, 8, 0, 4>("TMEM x4, 8 warps", nsm, out, cyc);
  run<1, 16, 0, 4>("TMEM x4, 16 warps", nsm, out, cyc);
  run<2, 0, 8, 16>("LDS.128, 8 warps", nsm, out, cyc);
  run<3, 8, 8, 16>("TMEM x16 8w + LDS.128 8w", nsm, out, cyc);
  run<3, 16, 8, 16>("TMEM x16 16w + LDS.128 8w", nsm, out, cyc);
  return 0;
}
