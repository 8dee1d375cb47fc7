// sweep2.cuh -- time-tiled (TK levels per pass) 3-D sweep for sm_100a, warp-specialised.
//
// The paper's method (time tiling; the CLooG schedule P:1437-1501) re-derived for
// a GPU (DESIGN.md §6 G2):
//   * one CTA owns a 64-column x GH-row x-y region and streams z;
//   * level l of the pass computes plane s - l*r while the TMA front is at plane s + r -- the
//     paper's skew of the time-tiled band by the stencil radius (P:1196-1202, P:1445
//     "int skew = 4*time"), applied to the streamed axis as a wavefront lag;
//   * the x-y region of level l shrinks by r per level (overlapped tiles: the redundant halo
//     work replaces the paper's sequential skewed tile order, which would serialise the SMs);
//   * only the last two levels (u^{n+TK-1}, u^{n+TK}) are written to HBM.
// Roles:
//   * warp NCW (producer): one lane TMA-loads every u^n plane box (region + r halo, out-of-bounds
//     zero fill = Dirichlet boundary) into a ring of mbarrier-tracked slots (full/empty);
//   * warps 0..NCW-1 (consumers): warp w owns rows [w*VY, (w+1)*VY) of the region at every level,
//     a column PAIR per lane (packed fp32x2).  Each level's z-column is a register queue of 2r+1
//     planes; the in-plane neighbours of level l >= 1 come from a shared-memory ring of level
//     l-1 planes with its own full/empty mbarriers (every consumer lane arrives).  No
//     __syncthreads in the steady state: warps drift within the ring depths.
//   * u^{n-1} and the medium of every level's plane are staged PD steps ahead with cp.async.
// Arithmetic is the canonical per-point order of include/stencil.h, so every value is
// bit-identical to the untiled sweep and to the CPU oracle (oracle/, never included here).
#pragma once
#include "sweep1.cuh"

namespace st {

template <int R, int TK, bool WAVE, int NCW, int VY>
struct Geom2 {
  static constexpr int RZ = R;                     // 3-D only
  static constexpr int QN = 2 * R + 1;
  static constexpr int RX2 = (R + 1) & ~1;
  static constexpr int RXB = (R + 3) & ~3;
  static constexpr int GW = 64;
  static constexpr int GH = NCW * VY;
  static constexpr int HX0 = Halo<R, TK>::hx(0);
  static constexpr int HY0 = R * (TK - 1);
  static constexpr int XS = HX0 % 4;               // keep the TMA box start 16-B aligned
  static constexpr int BW = GW + 2 * RXB + (XS ? 8 : 0);
  static constexpr int BH = GH + 2 * R;
  static constexpr int BCOL = RXB + XS;
  static constexpr int OX = GW - 2 * HX0;
  static constexpr int OY = GH - 2 * HY0;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
  static constexpr int DL = R + 3;                 // level-ring depth (planes); >= R + 1 needed
  static constexpr int LVL_F = GW * (GH + 2 * R);  // one level plane + R pad rows above/below
  static constexpr int LVL_BYTES = LVL_F * 4;
#ifndef ST_PD2
#define ST_PD2 2
#endif
  static constexpr int PD = ST_PD2;                // cp.async staging distance (steps)
  static constexpr int STAGE_F = WAVE ? VY * (64 + 128 * TK) : 0;   // prev + medium per level
  static constexpr int BAR_BYTES = 2048;
  static constexpr int FIXED_BYTES =
      BAR_BYTES + (TK - 1) * DL * LVL_BYTES + NCW * (PD + 1) * STAGE_F * 4;
  static constexpr int NTHREADS = 32 * (NCW + 1);
  static_assert(TK >= 2, "sweep2 is the time-tiled kernel");
  static_assert(OX > 0 && OY > 0, "tile too small for this radius / depth");
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
  static_assert(8 * (2 * 64 + 2 * (TK - 1) * DL) <= BAR_BYTES, "barrier area");
};

template <int R, int TK, bool WAVE, int NCW, int VY>
__global__ void __launch_bounds__(32 * (NCW + 1), 1)
sweep2_kernel(const __grid_constant__ CUtensorMap tmapC, const __grid_constant__ SweepParams p,
              const int nslot) {
  using G = Geom2<R, TK, WAVE, NCW, VY>;
  constexpr int QN = G::QN, RX2 = G::RX2, BW = G::BW, GW = G::GW, GH = G::GH, DL = G::DL;
  constexpr int HX0 = G::HX0, HY0 = G::HY0, BCOL = G::BCOL;
  constexpr int SLOT_F = G::SLOT_BYTES / 4, PD = G::PD, STAGE_F = G::STAGE_F;
  constexpr int NL = TK - 1;                        // levels with a shared-memory ring

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 64;
  uint64_t* lfull = empty + 64;                     // [NL][DL]
  uint64_t* lempty = lfull + NL * DL;               // [NL][DL]
  float* lring = reinterpret_cast<float*>(smem + G::BAR_BYTES);
  float* stage_all = lring + (size_t)NL * DL * G::LVL_F;
  float* ring = stage_all + (size_t)NCW * (PD + 1) * STAGE_F;   // 128-B aligned (sizes are)

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * G::OX, ty0 = blockIdx.y * G::OY;   // output tile origin
  const int gx = tx0 - HX0, gy = ty0 - HY0;                      // region origin
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;
  const int p_first = zb - TK * R;                  // first u^n plane (arrival 0)
  const int n_arr = (ze - zb) + 2 * TK * R;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 32 * NCW);
    }
    for (int i = 0; i < NL * DL; ++i) {
      mbar_init(&lfull[i], 32 * NCW);
      mbar_init(&lempty[i], 32 * NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ------------------------------------------------------------------ producer warp
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapC)) : "memory");
      int slot = 0;
      uint32_t ph = 0;
      for (int a = 0; a < n_arr; ++a) {
        if (a >= nslot) mbar_wait(&empty[slot], ph ^ 1u);
        mbar_expect_tx(&full[slot], (uint32_t)(BW * G::BH * 4));
        tma_load_3d(ring + (size_t)slot * SLOT_F, &tmapC, &full[slot], gx - BCOL, gy - R,
                    p_first + a - p.zv_lo);
        if (++slot == nslot) { slot = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  const int x0 = gx + 2 * lane;                     // my column pair
  const int ry = warp * VY;                         // my first region row
  const int y0 = gy + ry;                           // my first interior row
  const bool xin0 = (x0 >= 0) && (x0 < p.nx);
  const bool xin1 = (x0 + 1 >= 0) && (x0 + 1 < p.nx);
  const uint64_t xmask = (xin0 ? 0xffffffffull : 0ull) | (xin1 ? 0xffffffff00000000ull : 0ull);
  uint64_t rmask[VY];
  bool yin[VY];
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    yin[j] = (y0 + j >= 0) && (y0 + j < p.ny);
    rmask[j] = yin[j] ? xmask : 0ull;
  }
  bool any_row = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) any_row |= yin[j];
  const bool act = any_row && xin0;                 // this lane owns >= 1 interior point
  const uint64_t K0 = splat(p.K0);
  const uint64_t DT = splat(p.dt);
  // level l is computed on lanes [ex_l, 32-ex_l) and region rows [l*R, GH-l*R)
  // the last level's rows/lanes are the output tile
  const int ex_last = (HX0 - Halo<R, TK>::hx(TK - 1)) / 2;
  const bool lane_out = (lane >= ex_last) && (lane < 32 - ex_last);

  // rare events: does any of my rows hold a source (any level plane) / receiver (output planes)?
  bool wsrc = false, wrec = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    if (yin[j]) {
      const int zl = max(zb - (TK - 1) * R, p.gz_lo), zh = min(ze + (TK - 1) * R, p.gz_hi);
      if (zl < zh) wsrc |= row_has_entry(p.src_begin, p.src, zl, zh, y0 + j, gx, gx + 64);
      wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + j, tx0, tx0 + G::OX);
    }
  }
  wsrc = __any_sync(0xffffffffu, wsrc);
  wrec = __any_sync(0xffffffffu, wrec);

  // level l at arrival a computes plane a + p_first - (l+1)R, inside its range and the domain
  auto level_on = [&](int l, int a) -> bool {
    const int q = p_first + a - (l + 1) * R;
    return (q >= zb - (TK - 1 - l) * R) && (q < ze + (TK - 1 - l) * R) && (q >= p.gz_lo) &&
           (q < p.gz_hi);
  };

  // ---- staging of u^{n-1}(s) and the medium of every level's plane, PD steps ahead ----------
  const long long plane = p.plane;
  float* stage = stage_all + (size_t)warp * (PD + 1) * STAGE_F;
  const int rowoff = y0 * p.X + x0;                 // element offset of (first row, pair)
  const int X2 = p.X >> 1;
  const int acoff = y0 * X2 + (x0 >> 1);
  int a_iss = 0;                                    // next step to stage
  int e_iss = 0, e_use = 0;
  auto stage_next = [&]() {
    if (a_iss < n_arr && act) {
      float* e = stage + e_iss * STAGE_F;
      if (level_on(0, a_iss)) {
        const long long s = p_first + a_iss - R;
        const float* gP = p.P + s * plane + rowoff;
#pragma unroll
        for (int j = 0; j < VY; ++j)
          if (yin[j]) cp_async8(e + j * 64 + 2 * lane, gP + j * p.X);
      }
#pragma unroll
      for (int l = 0; l < TK; ++l) {
        if (level_on(l, a_iss)) {
          const long long q = p_first + a_iss - (l + 1) * R;
          const float4* gA = p.ac + q * (plane >> 1) + acoff;
#pragma unroll
          for (int j = 0; j < VY; ++j)
            if (yin[j]) cp_async16(e + VY * 64 + (l * VY + j) * 128 + 4 * lane, gA + j * X2);
        }
      }
    }
    cp_async_commit();
    ++a_iss;
    if (++e_iss == PD + 1) e_iss = 0;
  };
  if (WAVE) {
#pragma unroll 1
    for (int i = 0; i < PD; ++i) stage_next();
  }

  uint64_t qn[QN][VY];                              // u^n column queue (arrival-indexed)
  uint64_t ql[NL][QN][VY];                          // level l output queue, l = 0..TK-2
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) {
      qn[i][j] = 0ull;
#pragma unroll
      for (int l = 0; l < NL; ++l) ql[l][i][j] = 0ull;
    }

  int slot_a = 0;                                   // TMA ring slot of arrival a
  uint32_t ph_a = 0;
  int slot_c = R % nslot;                           // TMA ring slot of arrival a - R (centre);
                                                    // the first centre is arrival R (step 2R)
  int lslot_w = 0;                                  // level-ring slot written at step a
  uint32_t lph_w = 0;                               // parity of its previous use (empty wait)
  int lslot_r = 0;                                  // level-ring slot read at step a (plane a-R)
  uint32_t lph_r = 0;
  const int col = (ry + R) * BW + 2 * lane + BCOL;  // my first row, my pair, in a TMA slot
  const int lcol = (ry + R) * GW + 2 * lane;        // same in a level plane

  for (int base = 0; base < n_arr; base += QN) {
#pragma unroll
    for (int u = 0; u < QN; ++u) {
      const int a = base + u;
      if (a < n_arr) {
        // ---- arrival a: u^n plane p_first + a into the queue ----------------------------
        mbar_wait(&full[slot_a], ph_a);
        const float* sa = ring + slot_a * SLOT_F + col;
#pragma unroll
        for (int j = 0; j < VY; ++j) qn[u][j] = lds64(sa + j * BW);
        if (a < R) mbar_arrive(&empty[slot_a]);    // never a centre plane
        if (WAVE) stage_next();
        const float* st_e = stage + e_use * STAGE_F;
        if (WAVE && a >= 2 * R) cp_async_wait<PD>();   // this step's group has landed

        // ---- level 0 at plane s = p_first + a - R ---------------------------------------
        uint64_t out[VY];
#pragma unroll
        for (int j = 0; j < VY; ++j) out[j] = 0ull;
        if (a >= 2 * R) {                           // centre = arrival a - R >= R
          const int s = p_first + a - R;
          if (level_on(0, a)) {
            const float* rp0 = ring + slot_c * SLOT_F + col;
            uint64_t acc[VY];
            accumulate<R, R, QN, VY, 3, BW>(acc, qn, rp0, p, md<QN>(u - R));
            if (wsrc) {
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yin[j]) acc[j] = add_sources_row(acc[j], p, s, y0 + j, x0, p.wl_step);
            }
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c = qn[md<QN>(u - R)][j];
              uint64_t o;
              if (WAVE) {
                const uint64_t pv = lds64(st_e + j * 64 + 2 * lane);
                const float4 m4 = *reinterpret_cast<const float4*>(st_e + VY * 64 + j * 128 + 4 * lane);
                o = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c));
              } else {
                o = f2fma(DT, acc[j], c);
              }
              out[j] = o & rmask[j];
            }
            if (wrec && s >= zb && s < ze && lane_out) {
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yin[j] && ry + j >= HY0 && ry + j < GH - HY0)
                  sample_receivers_row(out[j], p, s, y0 + j, x0, p.tr_step);
            }
          }
          mbar_arrive(&empty[slot_c]);              // centre slot done (x/y neighbours read)
          if (++slot_c == nslot) slot_c = 0;
        }
#pragma unroll
        for (int j = 0; j < VY; ++j) ql[0][u][j] = out[j];

        // ---- levels 1..TK-1 ---------------------------------------------------------------
        // publish level 0 (plane s) into level-ring 0 slot lslot_w, then level l >= 1 reads the
        // ring of level l-1 at slot lslot_r (plane computed R steps ago).
#pragma unroll
        for (int l = 1; l < TK; ++l) {
          uint64_t* lf = lfull + (l - 1) * DL;
          uint64_t* le = lempty + (l - 1) * DL;
          float* lr = lring + (size_t)(l - 1) * DL * G::LVL_F;
          // publish level l-1 output of this step
          if (a >= DL) mbar_wait(&le[lslot_w], lph_w ^ 1u);
          {
            float* dst = lr + (size_t)lslot_w * G::LVL_F + lcol;
#pragma unroll
            for (int j = 0; j < VY; ++j) sts64(dst + j * GW, ql[l - 1][u][j]);
          }
          mbar_arrive(&lf[lslot_w]);
          // level l at plane q = p_first + a - (l+1)R: neighbours from the level-(l-1) plane
          // published R steps ago
          uint64_t ol[VY];
#pragma unroll
          for (int j = 0; j < VY; ++j) ol[j] = 0ull;
          if (a >= R) {
            mbar_wait(&lf[lslot_r], lph_r);
            const int q = p_first + a - (l + 1) * R;
            const int exl = (HX0 - Halo<R, TK>::hx(l)) / 2;
            const int eyl = l * R;
            const bool lane_in = (lane >= exl) && (lane < 32 - exl);
            const bool rows_in = (ry + VY > eyl) && (ry < GH - eyl);     // warp-uniform
            if (level_on(l, a) && rows_in) {
              const float* rp = lr + (size_t)lslot_r * G::LVL_F + lcol;
              uint64_t acc[VY];
              accumulate<R, R, QN, VY, 3, GW>(acc, ql[l - 1], rp, p, md<QN>(u - R));
              if (wsrc) {
#pragma unroll
                for (int j = 0; j < VY; ++j)
                  if (yin[j]) acc[j] = add_sources_row(acc[j], p, q, y0 + j, x0, p.wl_step + l);
              }
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                const uint64_t c = ql[l - 1][md<QN>(u - R)][j];
                uint64_t o;
                if (WAVE) {
                  const uint64_t pv = (l == 1) ? qn[md<QN>(u - 2 * R)][j]
                                               : ql[l >= 2 ? l - 2 : 0][md<QN>(u - 2 * R)][j];
                  const float4 m4 =
                      *reinterpret_cast<const float4*>(st_e + VY * 64 + (l * VY + j) * 128 + 4 * lane);
                  o = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c));
                } else {
                  o = f2fma(DT, acc[j], c);
                }
                const int rr = ry + j;
                ol[j] = (lane_in && rr >= eyl && rr < GH - eyl) ? (o & rmask[j]) : 0ull;
              }
              if (l == TK - 1) {
                // ---- last level: u^{n+TK} and u^{n+TK-1} on the output tile ------------------
                if (q >= zb && q < ze && lane_out && xin0) {
                  const long long off = (long long)q * plane + rowoff;
#pragma unroll
                  for (int j = 0; j < VY; ++j) {
                    const int rr = ry + j;
                    if (rr >= HY0 && rr < GH - HY0 && yin[j]) {
                      const uint64_t pv = ql[TK - 2][md<QN>(u - R)][j];
                      if (xin1) {
                        sts64(p.outC + off + j * p.X, ol[j]);
                        if (WAVE || p.write_prev) sts64(p.outP + off + j * p.X, pv);
                      } else {
                        p.outC[off + j * p.X] = lo_of(ol[j]);
                        if (WAVE || p.write_prev) p.outP[off + j * p.X] = lo_of(pv);
                      }
                    }
                  }
                }
              }
              if (wrec && q >= zb && q < ze && lane_out) {
#pragma unroll
                for (int j = 0; j < VY; ++j)
                  if (yin[j] && ry + j >= HY0 && ry + j < GH - HY0)
                    sample_receivers_row(ol[j], p, q, y0 + j, x0, p.tr_step + l);
              }
            }
            mbar_arrive(&le[lslot_r]);
          }
          if (l < TK - 1) {
#pragma unroll
            for (int j = 0; j < VY; ++j) ql[l < NL ? l : 0][u][j] = ol[j];
          }
        }
        // advance ring counters (the level rings of every level share the step schedule)
        if (++lslot_w == DL) { lslot_w = 0; lph_w ^= 1u; }
        if (a >= R) { if (++lslot_r == DL) { lslot_r = 0; lph_r ^= 1u; } }
        if (WAVE && ++e_use == PD + 1) e_use = 0;
        if (++slot_a == nslot) { slot_a = 0; ph_a ^= 1u; }
      }
    }
  }
  if (WAVE) cp_async_wait<0>();
}

}  // namespace st
