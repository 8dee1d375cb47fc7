// resident.cuh -- whole-run 2-D sweep resident in on-chip memory of one thread-block cluster
// (G4).
//
// For 2-D grids small enough to live in shared memory (BASELINE C1: 128 x 128 heat, 20 steps) the
// untiled sweep is launch-bound: 20 launches of 16 K points.  Temporal blocking taken to its end
// (keep computing further time levels while the data is on chip): a cluster of up to
// 8 CTAs splits the rows, each CTA loads its rows (+ an H = r*spb row halo) once and advances all
// nt steps in shared memory -- two time-level buffers, zero halo at the global boundary
// (Dirichlet); every spb steps each CTA pushes its H first / last rows straight into the
// neighbour CTAs' halo rows through distributed shared memory between two cluster barriers;
// in between the halo rows are recomputed redundantly (the paper's ghost zone of depth r*T_c).
// At the end it writes u^{n+nt-1}, u^{n+nt} back.  Same canonical per-point order as every other kernel
// (include/stencil.h), packed fp32x2 over column pairs, each thread a vertical strip of S rows
// whose y neighbours stay in registers; a bitmap of source column pairs routes the (rare) source
// points through the injection (acc += w in source index order, before the update); receivers are
// sampled from shared memory after each step.  The wave's u^{n+1} overwrites u^{n-1} in place
// (each pair reads only its own u^{n-1}), heat ping-pongs.
#pragma once
#include <cooperative_groups.h>

#include "sweep.cuh"

namespace st {

#ifndef ST_RES_THREADS
#define ST_RES_THREADS 512
#endif
constexpr int RES_THREADS = ST_RES_THREADS;
#ifndef ST_RES_CLUSTER
#define ST_RES_CLUSTER 16
#endif
constexpr int RES_CLUSTER = ST_RES_CLUSTER;   // CTAs per cluster (16: B200's non-portable maximum)
#ifndef ST_RES_STRIP
#define ST_RES_STRIP 2
#endif
constexpr int RES_STRIP = ST_RES_STRIP;   // rows per thread item (y neighbours reused from registers)

// padded row width: even left halo (8-byte aligned column pairs), right halo, even total
__host__ __device__ constexpr int res_left(int R) { return (R + 1) & ~1; }
__host__ __device__ inline int res_pitch(int R, int nx) { return (res_left(R) + nx + R + 1) & ~1; }
// rows owned by one CTA of a cluster of cs CTAs
__host__ __device__ inline int res_own(int ny, int cs) { return (ny + cs - 1) / cs; }
// rows per buffer: own rows + the H = r*spb halo on both sides, + a strip of slack
__host__ __device__ inline int res_rows(int R, int ny, int cs, int spb) {
  return res_own(ny, cs) + 2 * R * spb + RES_STRIP;
}
__host__ __device__ inline size_t res_smem_bytes(int R, bool wave, int nx, int ny, int cs, int spb) {
  const int rows = res_rows(R, ny, cs, spb);
  const size_t field = (size_t)res_pitch(R, nx) * rows * 4;
  const size_t medium = wave ? (size_t)((nx + 1) & ~1) * rows * 8 : 0;   // a, c incl. halo rows
  const size_t flags = ((size_t)((nx + 1) >> 1) * rows + 31) / 32 * 4;   // source-pair bitmap
  return 2 * field + medium + flags;
}
// cluster size: as many CTAs (<= cap) as keep >= r own rows each
__host__ __device__ inline int res_cluster(int R, int ny, int cap = RES_CLUSTER) {
  int cs = cap;
  while (cs > 1 && (res_own(ny, cs) < R || (cs - 1) * res_own(ny, cs) >= ny)) --cs;
  return cs;
}
// steps per cluster barrier: the halo H = r*spb must come from the two neighbours only
// (H <= own rows of every CTA but the last), at most 8
__host__ __device__ inline int res_spb(int R, int ny, int cs) {
  // measured on C1 (128^2 heat, 16 CTAs of 8 rows; bench GPts/s): spb 2/3/4/6/8 ->
  // 15.1/16.8/17.7/18.3/16.5 -- beyond 6 the redundant halo rows cost more than the barriers save
  if (cs == 1) return 8;
  int spb = 1;
  while (spb < 6 && R * (spb + 1) <= res_own(ny, cs)) ++spb;
  return spb;
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

// One step of a vertical strip of S rows of one column pair: the S + 2R pairs of the strip's
// column (centre + y neighbours) are loaded once into registers, x neighbours come from shared
// memory, the canonical accumulation runs per row (include/stencil.h), results are stored to `out`.
// b0: buffer row of the strip's first row; y0: its global row; rows >= yend are skipped.
template <int R, bool WAVE, int S>
__device__ __forceinline__ void res_strip(const float* C, float* out, const float* Am,
                                          const float* Cm, int pitch, int nx2, int x, int b0,
                                          int y0, int yend, int HL, const SweepParams& p,
                                          const unsigned* sflag, int pr, long long wl, bool xlast) {
  uint64_t col[S + 2 * R];
  const int i0 = b0 * pitch + HL + x;
#pragma unroll
  for (int j = 0; j < S + 2 * R; ++j) col[j] = lds64(C + i0 + (j - R) * pitch);
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int y = y0 + j;
    if (y >= yend) continue;   // (a `break` here faulted on sm_100a)
    const int i = i0 + j * pitch;
    const uint64_t c = col[j + R];
    uint64_t a = f2mul(splat(p.K0), c);
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      uint64_t sx;
      if ((k & 1) == 0) sx = f2add(lds64(C + i - k), lds64(C + i + k));
      else sx = pack2(fadd_ftz(C[i - k], C[i + k]), fadd_ftz(C[i + 1 - k], C[i + 1 + k]));
      a = f2fma(splat(p.W[0][k]), sx, a);
      a = f2fma(splat(p.W[1][k]), f2add(col[j + R - k], col[j + R + k]), a);
    }
    const int t = (b0 + j) * pr + (x >> 1);
    if ((sflag[t >> 5] >> (t & 31)) & 1u) a = res_sources(a, p, x, y, wl);
    uint64_t o;
    if (WAVE) {
      const int mi = (b0 + j) * nx2 + x;
      const uint64_t pv = lds64(out + i);              // u^{n-1}: overwritten in place below
      o = f2fma(pack2(Cm[mi], Cm[mi + 1]), a, f2fma(pack2(Am[mi], Am[mi + 1]), f2sub(pv, c), c));
    } else {
      o = f2fma(splat(p.dt), a, c);
    }
    if (xlast) o &= 0xffffffffull;                      // padding column stays zero
    sts64(out + i, o);
  }
}

// Cluster of cs CTAs (cluster dims (cs,1,1), grid (cs,1,1)); u_prev / u_cur in the library layout
// (outputs; the initial pair is read from in_prev / in_cur, which may be u_prev / u_cur -- no
// __restrict__: every CTA loads its rows before the first cluster barrier and stores after it)
// (2-D: one plane, row pitch p.X).  Every spb steps the CTAs exchange an H = r*spb row halo (the
// paper's ghost zone of depth r*T_c, here between the CTAs of a cluster) and
// recompute it redundantly in between (rows shrinking by r per step), so one cluster barrier
// serves spb steps.
template <int R, bool WAVE>
__global__ void __launch_bounds__(RES_THREADS, 1)
resident2d_kernel(const __grid_constant__ SweepParams p, float* u_prev, float* u_cur,
                  const float* in_prev, const float* in_cur, int nt, int spb) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) float sm[];
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int nx = p.nx, ny = p.ny, X = p.X;
  const int HL = res_left(R);
  const int pitch = res_pitch(R, nx);
  const int own = res_own(ny, cs);
  const int r0 = min(ny, rank * own), r1 = min(ny, r0 + own);   // my global rows [r0, r1)
  const int nrow = r1 - r0;
  const int H = R * spb;                                          // halo rows per side
  const int rows = res_rows(R, ny, cs, spb);
  const int fsz = pitch * rows;
  // buffer row b holds local row lr = b - H (global row r0 + lr)
  float* B0 = sm;                 // heat: ping-pong; wave: u^{n-1} (overwritten by u^{n+1})
  float* B1 = sm + fsz;           // u^n
  const int nx2 = (nx + 1) & ~1;
  float* Am = sm + 2 * fsz;       // wave: a, c per point of every buffer row (row pitch nx2)
  float* Cm = Am + nx2 * rows;
  const int pr = (nx + 1) >> 1;
  unsigned* sflag = reinterpret_cast<unsigned*>(sm + 2 * fsz + (WAVE ? 2 * nx2 * rows : 0));
  const int tid = threadIdx.x;

  // own shared memory first (nothing a predecessor grid writes), then wait for the predecessor
  for (int i = tid; i < 2 * fsz; i += RES_THREADS) sm[i] = 0.f;   // zero halo = Dirichlet
  for (int i = tid; i < (pr * rows + 31) / 32; i += RES_THREADS) sflag[i] = 0u;
  pdl_prologue_done();
  __syncthreads();
  // u^n, u^{n-1} (wave) and a, c (wave): own rows + the halo rows inside the grid
  const int lo = max(0, r0 - H), hi = min(ny, r1 + H);
  for (int i = tid; i < (hi - lo) * nx; i += RES_THREADS) {
    const int yy = i / nx, x = i - yy * nx;
    const int y = lo + yy;
    const int s = (y - r0 + H) * pitch + HL + x;
    B1[s] = in_cur[(size_t)y * X + x];
    if (WAVE) B0[s] = in_prev[(size_t)y * X + x];
  }
  if (WAVE) {
    const int X2 = X >> 1;
    for (int i = tid; i < pr * (hi - lo); i += RES_THREADS) {
      const int yy = i / pr, xp = i - yy * pr;
      const int b = lo + yy - r0 + H;
      const float4 m = p.ac[(size_t)(lo + yy) * X2 + xp];
      Am[b * nx2 + 2 * xp] = m.x; Am[b * nx2 + 2 * xp + 1] = m.y;
      Cm[b * nx2 + 2 * xp] = m.z; Cm[b * nx2 + 2 * xp + 1] = m.w;
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = p.src_begin[0]; q < p.src_begin[1]; ++q) {
      const int4 e = p.src[q];
      if (e.y < lo || e.y >= hi) continue;          // sources in the halo are injected there too
      const int t = (e.y - r0 + H) * pr + (e.x >> 1);
      sflag[t >> 5] |= 1u << (t & 31);
    }
  }
  const int rb = p.rec_begin[0], re = p.rec_begin[1];
  // neighbours' buffers (DSMEM): my first H rows go to the upper neighbour's bottom halo, my
  // last H rows to the lower neighbour's top halo (every CTA but the last owns >= H rows)
  const bool has_up = rank > 0 && nrow > 0, has_dn = r1 < ny && nrow > 0;
  float* up0 = has_up ? cluster.map_shared_rank(B0, rank - 1) : nullptr;
  float* dn0 = has_dn ? cluster.map_shared_rank(B0, rank + 1) : nullptr;
  cluster.sync();

  constexpr int S = RES_STRIP;
  const bool fixed_map = RES_THREADS % pr == 0;
  const int xp0 = tid % pr, sj0 = tid / pr, sstep = RES_THREADS / pr;
  float* cur = B1;
  float* oth = B0;
  int off = 0;                                   // oth - B0 (same offset in every CTA)
  for (int n = 0; n < nt;) {
    const int steps = min(spb, nt - n);
    for (int j = 0; j < steps; ++j, ++n) {
      const long long wl = p.wl_step + n;
      // local rows of this sub-step: the halo shrinks by r per step, never outside the grid
      const int ext = R * (steps - 1 - j);
      const int lr0 = max(-ext, -r0), lr1 = min(nrow + ext, ny - r0);
      // thread -> (column pair xp0, first strip sj0), then strips sj0 + k*sstep (no division in
      // the loop when the threads cover whole rows of pairs)
      const int nstr = (lr1 - lr0 + S - 1) / S;
      if (fixed_map) {
        for (int sj = sj0; sj < nstr; sj += sstep) {
          const int lr = lr0 + sj * S;
          res_strip<R, WAVE, S>(cur, oth, Am, Cm, pitch, nx2, 2 * xp0, lr + H, r0 + lr, r0 + lr1, HL,
                                p, sflag, pr, wl, 2 * xp0 + 1 >= nx);
        }
      } else {
        for (int t = tid; t < pr * nstr; t += RES_THREADS) {
          const int sj = t / pr, xp = t - sj * pr;
          const int lr = lr0 + sj * S;
          res_strip<R, WAVE, S>(cur, oth, Am, Cm, pitch, nx2, 2 * xp, lr + H, r0 + lr, r0 + lr1, HL,
                                p, sflag, pr, wl, 2 * xp + 1 >= nx);
        }
      }
      __syncthreads();
      for (int k = rb + tid; k < re; k += RES_THREADS) {
        const int4 e = p.rec[k];
        if (e.y >= r0 && e.y < r1)
          p.trace[(long long)(p.tr_step + n) * p.tr_stride + e.w] = oth[(e.y - r0 + H) * pitch + HL + e.x];
      }
      float* t_ = cur; cur = oth; oth = t_;
      off = fsz - off;
    }
    if (n < nt) {
      // halo push through distributed shared memory: u^n (cur) and, for the wave, u^{n-1} (oth).
      // First every CTA must be done reading its halo rows of this block (a neighbour's push
      // lands in them), then the pushes must land before the next block reads them.
      cluster.sync();
      const int coff = fsz - off;                    // cur - B0
      for (int i = tid; i < H * pitch; i += RES_THREADS) {
        const int rr = i / pitch, xx = i - rr * pitch;
        if (has_up) {
          up0[coff + (H + own + rr) * pitch + xx] = cur[(H + rr) * pitch + xx];
          if (WAVE) up0[off + (H + own + rr) * pitch + xx] = oth[(H + rr) * pitch + xx];
        }
        if (has_dn) {
          dn0[coff + rr * pitch + xx] = cur[(nrow + rr) * pitch + xx];
          if (WAVE) dn0[off + rr * pitch + xx] = oth[(nrow + rr) * pitch + xx];
        }
      }
      cluster.sync();
    }
  }
  __syncthreads();
  // write back own rows: u_cur = u^{n+nt}, u_prev = u^{n+nt-1}
  for (int i = tid; i < nrow * nx; i += RES_THREADS) {
    const int yy = i / nx, x = i - yy * nx;
    const int s = (yy + H) * pitch + HL + x;
    u_cur[(size_t)(r0 + yy) * X + x] = cur[s];
    u_prev[(size_t)(r0 + yy) * X + x] = oth[s];
  }
}

}  // namespace st
