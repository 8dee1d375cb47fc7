// Micro-benchmark: which data paths share the 128 B/clk/SM shared-memory crossbar on sm_100a?
//   LDS alone; LDG (L2-resident) alone; LDS + LDG; LDS + bulk copies L2 -> smem; LDS + STS.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub2 tools/ubench_smem_paths.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 2048;

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned ph) {
  unsigned ok = 0;
  do {
    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, q;\n\t}" : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  } while (!ok);
}

// MODE bits: 1 = LDS.64 x4 per iter (warps 0..NL-1), 2 = LDG.64 x4 per iter from an L2-resident
// buffer (same warps), 4 = one thread streams 16 KB bulk copies L2 -> smem (separate warp),
// 8 = STS.64 x2 per iter (same warps)
template <int MODE>
__global__ void __launch_bounds__(544, 1) kern(const float* __restrict__ g, size_t gfl, float* out,
                                               unsigned long long* cyc, unsigned long long* bytes_bulk,
                                               int zero) {
  extern __shared__ __align__(128) float sm[];   // 8192 floats for LDS + 2 x 16 KB bulk slots
  __shared__ __align__(8) unsigned long long bar[2];
  const int nl = 512;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i;
  if (threadIdx.x == 0) { mbar_init((unsigned)__cvta_generic_to_shared(&bar[0]), 1);
                          mbar_init((unsigned)__cvta_generic_to_shared(&bar[1]), 1);
                          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x >= nl) {
    if ((MODE & 4) && threadIdx.x == nl) {
      const long long t0 = clock64();
      unsigned long long nb = 0;
      const size_t chunk = 16384 / 4;
      for (int it = 0; it < 600; ++it) {
        const int s = it & 1;
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
        if (it >= 2) mbar_wait(b, ((it >> 1) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(16384) : "memory");
        const float* src = g + ((size_t)(blockIdx.x * 37 + it) * chunk) % (gfl - chunk);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"((unsigned)__cvta_generic_to_shared(sm + 8192 + s * 4096)), "l"(src), "r"(16384), "r"(b) : "memory");
        nb += 16384;
      }
      mbar_wait((unsigned)__cvta_generic_to_shared(&bar[0]), (299) & 1);
      mbar_wait((unsigned)__cvta_generic_to_shared(&bar[1]), (299) & 1);
      const long long t1 = clock64();
      bytes_bulk[blockIdx.x] = nb;
      cyc[1024 + blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    return;
  }
  float a0 = lane, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0, a6 = 0, a7 = 0;
  float c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + (w * 64 + lane * 2) * 4;
  const float2* gp = reinterpret_cast<const float2*>(g) + ((size_t)(blockIdx.x * 16 + w) * 4096 + lane) % (gfl / 2 - 8192);
  asm volatile("bar.sync 1, 512;" ::: "memory");
  const long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITER; ++it) {
    const unsigned off = ((it * 2048) & 16383) + (zero & it);
    if (MODE & 1) {
      float x, y;
#define L64(k, A, B)                                                                            \
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(base + off + k * 256)); \
  A += x; B += y;
      L64(0, a0, a1) L64(1, a2, a3) L64(2, a4, a5) L64(3, a6, a7)
    }
    if (MODE & 2) {
      const float2* q = gp + (size_t)((it * 128) & 2047);
#define G64(k, A, B) { float2 v; asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(q + k * 32)); A += v.x; B += v.y; }
      G64(0, c0, c1) G64(1, c2, c3) G64(2, c4, c5) G64(3, c6, c7)
    }
    if (MODE & 8) {
      asm volatile("st.shared.v2.f32 [%0], {%1,%2};" :: "r"(base + ((off + 8192) & 16383)), "f"(a0), "f"(c1) : "memory");
      asm volatile("st.shared.v2.f32 [%0], {%1,%2};" :: "r"(base + ((off + 12288) & 16383)), "f"(a2), "f"(c3) : "memory");
    }
  }
  const long long t1 = clock64();
  float r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
  if (r == 1234.5f) out[threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE>
void run(const char* name, int nsm, const float* g, size_t gfl, float* out, unsigned long long* cyc,
         unsigned long long* bb) {
  const int smem = 8192 * 4 + 2 * 16384;
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<MODE><<<nsm, 544, smem>>>(g, gfl, out, cyc, bb, 0);
  cudaDeviceSynchronize();
  kern<MODE><<<nsm, 544, smem>>>(g, gfl, out, cyc, bb, 0);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2048], hb[1024];
  cudaMemcpy(h, cyc, 2048 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, bb, nsm * 8, cudaMemcpyDeviceToHost);
  double c = 0, cb = 0, nb = 0;
  for (int i = 0; i < nsm; ++i) { c += h[i]; cb += h[1024 + i]; nb += hb[i]; }
  c /= nsm; cb /= nsm; nb /= nsm;
  const double per = c / ITER, warps = 16;
  printf("%-26s cyc/iter %7.2f  LDS %6.2f  LDG %6.2f  STS %6.2f B/clk/SM", name, per,
         (MODE & 1) ? warps * 1024 / per : 0.0, (MODE & 2) ? warps * 1024 / per : 0.0,
         (MODE & 8) ? warps * 512 / per : 0.0);
  if (MODE & 4) printf("  bulk %6.2f B/clk/SM over %.0f cyc", nb / cb, cb);
  printf("  (%s)\n", cudaGetErrorString(e));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t gfl = (size_t)16 << 20;   // 64 MB: L2-resident after the first pass
  float *g, *out; unsigned long long *cyc, *bb;
  cudaMalloc(&g, gfl * 4); cudaMemset(g, 0, gfl * 4);
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 2048 * 8); cudaMalloc(&bb, 1024 * 8);
  cudaMemset(cyc, 0, 2048 * 8); cudaMemset(bb, 0, 1024 * 8);
  run<1>("LDS", nsm, g, gfl, out, cyc, bb);
  run<2>("LDG (L2)", nsm, g, gfl, out, cyc, bb);
  run<3>("LDS + LDG", nsm, g, gfl, out, cyc, bb);
  run<4>("bulk only", nsm, g, gfl, out, cyc, bb);
  run<5>("LDS + bulk", nsm, g, gfl, out, cyc, bb);
  run<8>("STS", nsm, g, gfl, out, cyc, bb);
  run<9>("LDS + STS", nsm, g, gfl, out, cyc, bb);
  return 0;
}
