// sweeph.cuh -- time-tiled heat sweep (G5): all TK levels of a region in one warp's registers.
//
// The paper's time tile (skew by the radius P:1189-1202) for the diffusion stencil
// (P:487-556), laid out for the measured limit of the B200 SM: every LDS / SHFL byte crosses the
// same 128 B/clk/SM shared-memory crossbar (tools/ubench_smem_*.cu), while TMA
// writes into shared memory do not.  So each value stays in the register file of the thread that
// produced it for as long as possible:
//   * one CTA owns a 64-column x GH-row region (GH = NW*VY) and streams z; the output tile is the
//     region shrunk by HX (x, even) and HY = TK*r (y) on each side (overlapped tiles);
//   * the u^n planes arrive by TMA (region box, no halo, out-of-bounds zero fill) in a ring;
//   * warp w owns VY rows, lane a column PAIR (packed fp32x2).  At step a it computes EVERY level
//     l = 0..TK-1, level l at plane p_first + a - (l+1)r (the wavefront lag r per level): its z
//     neighbours are its own register queues (level l's queue holds level l-1's outputs), its x
//     neighbours come from the lanes beside it by SHFL, its y neighbours from its own rows and,
//     for the r rows beyond its strip, from the neighbour warps' boundary rows, which every warp
//     publishes per level and plane into a small shared-memory ring (STS of 2r of its VY rows);
//   * values that depend on data beyond the region (the x/y rim that shrinks by r per level) are
//     computed from whatever the edge lanes / clamped rows hold and never stored -- the output
//     tile only reads values whose dependence cone lies inside the region;
//   * one CTA barrier per step orders the boundary-row ring and the TMA ring: everything a warp
//     reads from another warp was written at least r steps earlier.
// Level l writes nothing to HBM except the last level (u^{n+TK}) and, on the last pass of a run,
// u^{n+TK-1}: HBM traffic 8/TK B per update.  Arithmetic is the canonical per-point order of
// include/stencil.h (bit-identical to the oracle, which is never included here).
#pragma once
#include "sweep2.cuh"
#include <type_traits>

namespace st {

#ifndef ST_H_STEADY
#define ST_H_STEADY 1
#endif

template <int R, int TK, int VY, int NW>
struct GeomH {
  static constexpr int GW = 64;
  static constexpr int GH = NW * VY;                // region rows
  static constexpr int QN = 2 * R + 1;              // z-queue length per level
  static constexpr int HX = (TK * R + 1) & ~1;      // x rim (even: column pairs never straddle it)
  static constexpr int HY = TK * R;                 // y rim
  static constexpr int OX = GW - 2 * HX;            // output tile (OX = 0 mod 4)
  static constexpr int OY = GH - 2 * HY;
  static constexpr int XS = HX % 4;                 // box starts XS columns left (16-B aligned)
  static constexpr int BW = GW + (XS ? 8 : 0);      // TMA box width (multiple of 8 floats)
  static constexpr int BH = GH;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
  static constexpr int D = R + 1;                   // boundary-row ring depth (planes)
  static constexpr int BND_ENTRY = 2 * R * GW * 4;  // one warp's r top + r bottom rows
  static constexpr int BAR_BYTES = 512;             // full barriers (<= 64 slots)
  static constexpr int BND_BYTES = (TK - 1) * D * NW * BND_ENTRY;
  static constexpr int FIXED_BYTES = (BAR_BYTES + BND_BYTES + 127) / 128 * 128;
  static constexpr int NTHREADS = 32 * NW;
  static_assert(VY >= R, "boundary rows come from the adjacent warp only");
  static_assert(OX > 0 && OY > 0, "tile too small for this radius / depth");
  static_assert(TK >= 2, "time-tiled instance");
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
};

// Column 2*lane + d of the packed pair c held by the lanes of the warp (d = 0, 1: own pair).
// Lanes beyond the warp return their own value: those columns lie in the rim (never stored).
template <int d>
__device__ __forceinline__ float col_of(uint64_t c) {
  if constexpr (d == 0) return lo_of(c);
  else if constexpr (d == 1) return hi_of(c);
  else {
    constexpr int m = (d >= 0) ? (d >> 1) : -((1 - d) >> 1);   // floor(d / 2)
    const float v = (d & 1) ? hi_of(c) : lo_of(c);
    if constexpr (m < 0) return __shfl_up_sync(0xffffffffu, v, -m);
    else return __shfl_down_sync(0xffffffffu, v, m);
  }
}

template <int R, int K = 1>
__device__ __forceinline__ void xsums(uint64_t (&sx)[R + 1], uint64_t c) {
  if constexpr (K <= R) {
    sx[K] = pack2(fadd_ftz(col_of<-K>(c), col_of<K>(c)), fadd_ftz(col_of<1 - K>(c), col_of<1 + K>(c)));
    xsums<R, K + 1>(sx, c);
  }
}

template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// MODE bit 0: SAVE (snapshot store of the last level), bit 1: EV (sources / receivers present).
// The plain instance (MODE 0) carries no event code in its step body.
template <int R, int TK, int VY, int NW, int MODE>
__global__ void __launch_bounds__(32 * NW, 1)
sweeph_kernel(const __grid_constant__ CUtensorMap tmapC, const __grid_constant__ SweepParams p,
              const int nslot) {
  constexpr bool SAVE = MODE & 1, EV = MODE & 2;
  using G = GeomH<R, TK, VY, NW>;
  constexpr int QN = G::QN, GW = G::GW, GH = G::GH, BW = G::BW, D = G::D;
  constexpr int HX = G::HX, HY = G::HY, SLOT = G::SLOT_BYTES, BE = G::BND_ENTRY;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * G::OX, ty0 = blockIdx.y * G::OY;   // output tile origin
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;                                             // CTA-uniform
  const int p_first = zb - TK * R;
  const int n_arr = (ze - zb) + 2 * TK * R;
  const int gx = tx0 - HX, gy = ty0 - HY;                           // region origin
  const uint32_t ring = sbase + G::FIXED_BYTES;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) mb_init(sbase + 8 * i, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_prologue_done();
  auto issue = [&](int b, int slot) {   // TMA of arrival b (plane p_first + b) into ring slot
    mb_expect_tx(sbase + 8 * slot, (uint32_t)(BW * GH * 4));
    tma_load_3d_s(ring + slot * SLOT, &tmapC, sbase + 8 * slot, gx - G::XS, gy, p_first + b - p.zv_lo);
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapC)) : "memory");
    for (int b = 0; b < nslot && b < n_arr; ++b) issue(b, b);
  }

  // ---- per-thread geometry
  const int x0 = gx + 2 * lane;
  const bool xin0 = (x0 >= 0) && (x0 < p.nx), xin1 = (x0 + 1 >= 0) && (x0 + 1 < p.nx);
  const uint64_t xmask = (xin0 ? 0xffffffffull : 0ull) | (xin1 ? 0xffffffff00000000ull : 0ull);
  const int wr = warp * VY;                          // my first region row
  const int y0 = gy + wr;
  unsigned smask = 0;                                // bit j: row j is an output row in the domain
  unsigned ymask = 0;                                // bit j: row j is in the domain
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    const bool yin = (y0 + j >= 0) && (y0 + j < p.ny);
    ymask |= yin ? (1u << j) : 0u;
    smask |= (yin && (wr + j >= HY) && (wr + j < GH - HY)) ? (1u << j) : 0u;
  }
  const bool lane_out = (lane >= HX / 2) && (lane < 32 - HX / 2) && xin0;
  if (!lane_out) smask = 0;
  // rare events (warp-uniform)
  bool wsrc = false, wrec = false;
  if (EV) {
    const int qlo0 = max(zb - (TK - 1) * R, p.gz_lo), qhi0 = min(ze + (TK - 1) * R, p.gz_hi);
#pragma unroll
    for (int j = 0; j < VY; ++j) {
      if ((ymask >> j) & 1) {
        if (qlo0 < qhi0) wsrc |= row_has_entry(p.src_begin, p.src, qlo0, qhi0, y0 + j, gx, gx + GW);
        if ((smask >> j) & 1) wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + j, tx0, tx0 + G::OX);
      }
    }
    wsrc = __any_sync(0xffffffffu, wsrc);
    wrec = __any_sync(0xffffffffu, wrec);
  }

  // shared-memory addresses (bytes)
  const uint32_t my_col = (G::XS + 2 * lane) * 4;
  const uint32_t own_off = wr * BW * 4 + my_col;                               // row wr of a slot
  const uint32_t up_off = max(wr - R, 0) * BW * 4 + my_col;                    // rows wr-R.. (clamped)
  const uint32_t dn_off = min(wr + VY, GH - R) * BW * 4 + my_col;              // rows wr+VY.. (clamped)
  const uint32_t bnd = sbase + G::BAR_BYTES;
  // boundary ring entry (level l, slot s, warp w): rows [top 0..R-1 | bottom 0..R-1] x 64 floats
  const uint32_t b_mine = bnd + warp * BE + 8 * lane;
  const uint32_t b_up = bnd + max(warp - 1, 0) * BE + R * GW * 4 + 8 * lane;       // its bottom rows
  const uint32_t b_dn = bnd + min(warp + 1, NW - 1) * BE + 8 * lane;                // its top rows
  const uint64_t DT = splat(p.dt), K0 = splat(p.K0);
  const long long plane = p.plane;
  const int X = p.X;
  // output pointer of the last level's plane at step a (advances by one plane per step);
  // u^{n+TK-1} and the snapshot live at fixed element distances from it
  float* oz = p.outC + (long long)(p_first - TK * R) * plane + (long long)y0 * X + x0;
  const long long dP = p.outP - p.outC, dS = SAVE ? p.outS - p.outC : 0;
  const bool wprev = p.write_prev != 0;
  // the region lies inside the domain: no level output needs the Dirichlet mask (CTA-uniform)
  const bool edge = !(gx >= 0 && gx + GW <= p.nx && gy >= 0 && gy + GH <= p.ny);

  // steady steps: every level's queue is full and its plane inside the global interior
  int st_lo = 2 * TK * R, st_hi = n_arr;
#pragma unroll
  for (int l = 0; l < TK; ++l) {
    st_lo = max(st_lo, max(zb - (TK - 1 - l) * R, p.gz_lo) - p_first + (l + 1) * R);
    st_hi = min(st_hi, min(ze + (TK - 1 - l) * R, p.gz_hi) - p_first + (l + 1) * R);
  }

  uint64_t q[TK][QN][VY];
#pragma unroll
  for (int l = 0; l < TK; ++l)
#pragma unroll
    for (int i = 0; i < QN; ++i)
#pragma unroll
      for (int j = 0; j < VY; ++j) q[l][i][j] = 0ull;

  int s_a = 0;  uint32_t ph_a = 0;        // ring slot / parity of arrival a
  int s_c = 0;                            // ring slot of arrival a - R (level-0 centre)
  int bw_ = 0;                            // boundary slot written at step a (a mod D)

  // one step (arrival a, queue index UU = a mod QN); CHECK: prologue / epilogue / boundary steps
  auto step = [&](auto CHK, auto EDG, auto UU, const int a) {
    constexpr bool CHECK = decltype(CHK)::value;
    constexpr bool EDGE = decltype(EDG)::value;
    constexpr int iN = decltype(UU)::value, iC = md<QN>(iN - R);
    if (CHECK && a >= n_arr) return;
    const int br = (bw_ + 1 == D) ? 0 : bw_ + 1;   // (a - R) mod D
    mb_wait(sbase + 8 * s_a, ph_a);
    {
      const uint32_t s = ring + s_a * SLOT + own_off;
#pragma unroll
      for (int j = 0; j < VY; ++j) q[0][iN][j] = ld_s64r(s + j * BW * 4);
    }
    static_for<0, TK>([&](auto LL) {
      constexpr int l = decltype(LL)::value;
      if (CHECK && a < 2 * (l + 1) * R) return;          // level l's queue not full yet
      const int z = p_first + a - (l + 1) * R;
      const bool act = !CHECK || (z >= max(zb - (TK - 1 - l) * R, p.gz_lo) &&
                                  z < min(ze + (TK - 1 - l) * R, p.gz_hi));
      uint64_t o[VY];
      if (act) {
        uint64_t up[R], dn[R];                            // y neighbours beyond the strip
        if constexpr (l == 0) {
          const uint32_t cs = ring + s_c * SLOT;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            up[i] = ld_s64r(cs + up_off + i * BW * 4);
            dn[i] = ld_s64r(cs + dn_off + i * BW * 4);
          }
        } else {
          const uint32_t e = ((l - 1) * D + br) * NW * BE;
#pragma unroll
          for (int i = 0; i < R; ++i) {
            up[i] = ld_s64r(e + b_up + i * GW * 4);
            dn[i] = ld_s64r(e + b_dn + i * GW * 4);
          }
        }
        uint64_t acc[VY];
#pragma unroll
        for (int j = 0; j < VY; ++j) {
          const uint64_t c = q[l][iC][j];
          uint64_t sx[R + 1];
          xsums<R>(sx, c);
          uint64_t a2 = f2mul(K0, c);
#pragma unroll
          for (int k = 1; k <= R; ++k) {
            a2 = f2fma(splat(p.W[0][k]), sx[k], a2);
            const uint64_t yl = (j - k >= 0) ? q[l][iC][(j - k) >= 0 ? j - k : 0] : up[(R + j - k) >= 0 ? R + j - k : 0];
            const uint64_t yr = (j + k < VY) ? q[l][iC][(j + k) < VY ? j + k : 0] : dn[(j + k - VY) >= 0 ? j + k - VY : 0];
            a2 = f2fma(splat(p.W[1][k]), f2add(yl, yr), a2);
            a2 = f2fma(splat(p.W[2][k]), f2add(q[l][md<QN>(iC - k)][j], q[l][md<QN>(iC + k)][j]), a2);
          }
          acc[j] = a2;
        }
        if (EV && wsrc) {
#pragma unroll
          for (int j = 0; j < VY; ++j)
            if ((ymask >> j) & 1) acc[j] = add_sources_row(acc[j], p, z, y0 + j, x0, p.wl_step + l);
        }
#pragma unroll
        for (int j = 0; j < VY; ++j) {
          o[j] = f2fma(DT, acc[j], q[l][iC][j]);
          if (EDGE) o[j] &= ((ymask >> j) & 1) ? xmask : 0ull;
        }
      } else {
#pragma unroll
        for (int j = 0; j < VY; ++j) o[j] = 0ull;
      }
      if constexpr (l < TK - 1) {
#pragma unroll
        for (int j = 0; j < VY; ++j) q[l + 1][iN][j] = o[j];
        // publish my top / bottom R rows of this level's plane
        const uint32_t e = (l * D + bw_) * NW * BE + b_mine;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          st_s64(e + i * GW * 4, o[i]);
          st_s64(e + (R + i) * GW * 4, o[VY - R + i]);
        }
      } else {
        // u^{n+TK} (and u^{n+TK-1} on the last pass) on the output tile
        if (act && smask) {
#pragma unroll
          for (int j = 0; j < VY; ++j) {
            if ((smask >> j) & 1) {
              float* d = oz + j * X;
              if (xin1) {
                sts64(d, o[j]);
                if (wprev) sts64(d + dP, q[l][iC][j]);
                if (SAVE) sts64(d + dS, o[j]);
              } else {
                d[0] = lo_of(o[j]);
                if (wprev) d[dP] = lo_of(q[l][iC][j]);
                if (SAVE) d[dS] = lo_of(o[j]);
              }
            }
          }
        }
      }
      if (EV && wrec && act && z >= zb && z < ze && smask) {
#pragma unroll
        for (int j = 0; j < VY; ++j)
          if ((smask >> j) & 1) sample_receivers_row(o[j], p, z, y0 + j, x0, p.tr_step + l);
      }
    });
    // every warp is done with step a: boundary rows of step a are visible to later steps,
    // the ring slot of arrival a - R (last read as level-0 centre) is free
    __syncthreads();
    if (!CHECK || a >= R) {   // refill the slot of arrival a - R with arrival a - R + nslot
      if (tid == 0 && a - R + nslot < n_arr) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(a - R + nslot, s_c);
      }
      if (++s_c == nslot) s_c = 0;
    }
    if (++s_a == nslot) { s_a = 0; ph_a ^= 1u; }
    if (++bw_ == D) bw_ = 0;
    oz += plane;
  };

  // ST_H_STEADY: compile a check-free step body for the steady blocks (1) or run every block with
  // the uniform level/plane checks (0: half the code; the kernel is instruction-cache bound at
  // T_k = 4 with 6-row strips, ncu no_instruction stalls)
  auto run = [&](auto EDG) {
#pragma unroll 1
    for (int base = 0; base < n_arr; base += QN) {
      if (ST_H_STEADY && base >= st_lo && base + QN <= st_hi) {
        static_for<0, QN>([&](auto UU) { step(std::false_type{}, EDG, UU, base + decltype(UU)::value); });
      } else {
        static_for<0, QN>([&](auto UU) { step(std::true_type{}, EDG, UU, base + decltype(UU)::value); });
      }
    }
  };
#ifndef ST_H_EDGE_SPLIT
#define ST_H_EDGE_SPLIT 1   // 0: one body that always applies the Dirichlet mask (half the code)
#endif
  if (edge || !ST_H_EDGE_SPLIT) run(std::true_type{});
  else run(std::false_type{});
}

}  // namespace st
