// resident.cuh -- whole-run 2-D sweep resident in shared memory (G4).
//
// For 2-D grids small enough to live in one SM's shared memory (BASELINE C1: 128 x 128 heat, 20
// steps) the untiled sweep is launch-bound: 20 launches of 16 K points.  Temporal blocking taken
// to its end (keep computing further time levels while the data is on chip): one CTA
// loads the interior once, advances all nt steps in shared memory (zero halo = Dirichlet, two
// time-level buffers, __syncthreads between steps) and writes u^{n+nt-1}, u^{n+nt} back.  Same
// canonical per-point order as every other kernel (include/stencil.h), packed fp32x2 over column
// pairs; a bitmap of source column pairs routes the (rare) source points through the injection
// (acc += w in source index order, before the update); receivers are sampled from shared memory
// after each step.  The wave's u^{n+1} overwrites u^{n-1} in place (each pair reads only its own
// u^{n-1}), heat ping-pongs.
#pragma once
#include "sweep.cuh"

namespace st {

constexpr int RES_THREADS = 1024;

// padded row width: even left halo (8-byte aligned column pairs), right halo, even total
__host__ __device__ constexpr int res_left(int R) { return (R + 1) & ~1; }
__host__ __device__ inline int res_pitch(int R, int nx) { return (res_left(R) + nx + R + 1) & ~1; }
__host__ __device__ inline size_t res_smem_bytes(int R, bool wave, int nx, int ny) {
  const size_t field = (size_t)res_pitch(R, nx) * (ny + 2 * R) * 4;
  const size_t medium = wave ? (size_t)((nx + 1) & ~1) * ny * 8 : 0;   // a, c per point
  const size_t flags = ((size_t)((nx + 1) >> 1) * ny + 31) / 32 * 4;   // source-pair bitmap
  return 2 * field + medium + flags;
}

// sources at (x or x+1, y), in index order per element: acc += w (canonical position)
__device__ __noinline__ uint64_t res_sources(uint64_t a, const SweepParams& p, int x, int y,
                                             long long wl) {
  const int sb = p.src_begin[0], se = p.src_begin[1];
  for (int q = sb; q < se; ++q) {
    const int4 e = p.src[q];
    if (e.y != y) continue;
    const float w = p.wavelet[wl * p.wl_stride + e.w];
    if (e.x == x) a = pack2(fadd_ftz(lo_of(a), w), hi_of(a));
    else if (e.x == x + 1) a = pack2(lo_of(a), fadd_ftz(hi_of(a), w));
  }
  return a;
}

template <int R, bool WAVE>
__device__ __forceinline__ uint64_t res_update(const float* C, const float* P, const float* A,
                                               const float* Cm, int pitch, int i, int mi,
                                               const SweepParams& p, bool src, int x, int y,
                                               long long wl) {
  // i: index of the pair's left point in the padded buffers; mi: in the a/c arrays
  const uint64_t c = lds64(C + i);
  uint64_t a = f2mul(splat(p.K0), c);
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    uint64_t sx;
    if ((k & 1) == 0) {
      sx = f2add(lds64(C + i - k), lds64(C + i + k));
    } else {
      sx = pack2(fadd_ftz(C[i - k], C[i + k]), fadd_ftz(C[i + 1 - k], C[i + 1 + k]));
    }
    a = f2fma(splat(p.W[0][k]), sx, a);
    a = f2fma(splat(p.W[1][k]), f2add(lds64(C + i - k * pitch), lds64(C + i + k * pitch)), a);
  }
  if (src) a = res_sources(a, p, x, y, wl);
  if (WAVE) {
    const uint64_t pv = lds64(P + i);
    const uint64_t av = pack2(A[mi], A[mi + 1]), cv = pack2(Cm[mi], Cm[mi + 1]);
    return f2fma(cv, a, f2fma(av, f2sub(pv, c), c));
  }
  return f2fma(splat(p.dt), a, c);
}

// One CTA; u_prev / u_cur in the library layout (2-D: one plane, row pitch p.X).
template <int R, bool WAVE>
__global__ void __launch_bounds__(RES_THREADS, 1)
resident2d_kernel(const __grid_constant__ SweepParams p, float* __restrict__ u_prev,
                  float* __restrict__ u_cur, int nt) {
  extern __shared__ __align__(16) float sm[];
  const int nx = p.nx, ny = p.ny, X = p.X;
  const int HL = res_left(R);
  const int pitch = res_pitch(R, nx);
  const int rows = ny + 2 * R;
  const int fsz = pitch * rows;
  float* B0 = sm;                 // heat: ping-pong; wave: u^{n-1} (overwritten by u^{n+1})
  float* B1 = sm + fsz;           // wave: u^n
  const int nx2 = (nx + 1) & ~1;
  float* Am = sm + 2 * fsz;       // wave: a, c per point (row pitch nx2)
  float* Cm = Am + nx2 * ny;
  const int tid = threadIdx.x;

  pdl_prologue_done();
  // zero both buffers (halo = Dirichlet), then load the interior
  for (int i = tid; i < 2 * fsz; i += RES_THREADS) sm[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < nx * ny; i += RES_THREADS) {
    const int y = i / nx, x = i - y * nx;
    const int s = (y + R) * pitch + HL + x;
    B1[s] = u_cur[(size_t)y * X + x];
    if (WAVE) B0[s] = u_prev[(size_t)y * X + x];
  }
  if (WAVE) {
    const int X2 = X >> 1;
    for (int i = tid; i < (nx2 >> 1) * ny; i += RES_THREADS) {
      const int y = i / (nx2 >> 1), xp = i - y * (nx2 >> 1);
      const float4 m = p.ac[(size_t)y * X2 + xp];
      Am[y * nx2 + 2 * xp] = m.x; Am[y * nx2 + 2 * xp + 1] = m.y;
      Cm[y * nx2 + 2 * xp] = m.z; Cm[y * nx2 + 2 * xp + 1] = m.w;
    }
  }
  __syncthreads();

  // sources / receivers of the (single) plane, from the per-plane tables; a bitmap marks the
  // column pairs that hold a source
  const int rb = p.rec_begin[0], re = p.rec_begin[1];
  const int pr = (nx + 1) >> 1;
  const int npairs = pr * ny;
  unsigned* sflag = reinterpret_cast<unsigned*>(Cm + (WAVE ? nx2 * ny : 0));
  for (int i = tid; i < (npairs + 31) / 32; i += RES_THREADS) sflag[i] = 0u;
  __syncthreads();
  if (tid == 0) {
    for (int q = p.src_begin[0]; q < p.src_begin[1]; ++q) {
      const int4 e = p.src[q];
      const int t = e.y * pr + (e.x >> 1);
      sflag[t >> 5] |= 1u << (t & 31);
    }
  }
  __syncthreads();
  float* cur = B1;                // u^n
  float* oth = B0;                // heat: scratch; wave: u^{n-1}, overwritten in place by u^{n+1}
  for (int n = 0; n < nt; ++n) {
    const long long wl = p.wl_step + n;
    for (int t = tid; t < npairs; t += RES_THREADS) {
      const int y = t / pr, xp = t - y * pr;
      const int x = 2 * xp;
      const int i = (y + R) * pitch + HL + x;
      const bool src = (sflag[t >> 5] >> (t & 31)) & 1u;
      uint64_t o = res_update<R, WAVE>(cur, oth, Am, Cm, pitch, i, y * nx2 + x, p, src, x, y, wl);
      if (x + 1 >= nx) o &= 0xffffffffull;              // padding column stays zero
      sts64(oth + i, o);
    }
    __syncthreads();
    for (int k = rb + tid; k < re; k += RES_THREADS) {
      const int4 e = p.rec[k];
      p.trace[(long long)(p.tr_step + n) * p.tr_stride + e.w] = oth[(e.y + R) * pitch + HL + e.x];
    }
    float* t_ = cur; cur = oth; oth = t_;
  }
  __syncthreads();
  // write back: u_cur = u^{n+nt}, u_prev = u^{n+nt-1}
  for (int i = tid; i < nx * ny; i += RES_THREADS) {
    const int y = i / nx, x = i - y * nx;
    const int s = (y + R) * pitch + HL + x;
    u_cur[(size_t)y * X + x] = cur[s];
    u_prev[(size_t)y * X + x] = oth[s];
  }
}

}  // namespace st
