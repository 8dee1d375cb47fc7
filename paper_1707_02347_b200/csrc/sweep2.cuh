// sweep2.cuh -- time-tiled (TK levels per pass) 3-D sweep for sm_100a: one warp group per level.
//
// The paper's method (time tiling; the CLooG schedule P:1437-1501) re-derived for
// a GPU (DESIGN.md §6 G2):
//   * one CTA owns a 64-column x GH-row x-y region (GH = OY + 2r(TK-1)) and streams z;
//   * at step a, level l computes plane p_first + a - (l+1)r: each level trails the one below it
//     by r planes -- the paper's skew of the time-tiled band by the stencil radius (P:1196-1202,
//     P:1445 "int skew = 4*time"), applied to the streamed axis as a wavefront lag;
//   * the x-y region shrinks by r per level (overlapped tiles: the redundant halo work replaces
//     the paper's sequential skewed tile order, which would serialise the SMs);
//   * only the last two levels (u^{n+TK-1}, u^{n+TK}) of the output tile are written to HBM.
// Roles (a software pipeline across warp groups, no __syncthreads in the steady state):
//   * warp NCW (producer): one lane TMA-loads every u^n plane box (region + r halo, out-of-bounds
//     zero fill = Dirichlet boundary) into a ring of mbarrier-tracked slots (full/empty);
//   * group l (warps(l) warps, two rows each, a column PAIR per lane, packed fp32x2) computes
//     level l.  Its input planes come from the TMA ring (l = 0) or from the shared-memory ring of
//     level l-1 (each slot guarded by a full/empty mbarrier pair); it keeps the z-column of its
//     rows in a register queue of 2r+1 planes and takes the x/y neighbours from the centre plane
//     in shared memory.  Levels below TK-1 publish every plane into their own ring; the last
//     level writes u^{n+TK}, u^{n+TK-1} to global memory.
//   * the producer also streams, per step, u^{n-1} and the medium of level 0's plane and u^n and
//     the medium of level 1's plane (wave) as TMA boxes into two more mbarrier rings, so the
//     consumer warps never touch global memory except for the final stores.
// All shared-memory traffic uses 32-bit shared-window addresses.  Arithmetic is the canonical
// per-point order of include/stencil.h, so every value is bit-identical to the untiled sweep and
// to the CPU oracle (oracle/, never included here).
#pragma once
#include "sweep1.cuh"

namespace st {

// ------------------------------------------------------------ 32-bit shared-window primitives
template <int OFF>
__device__ __forceinline__ uint64_t ld_s64(uint32_t a) {
  uint64_t v; asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(OFF)); return v;
}
__device__ __forceinline__ uint64_t ld_s64r(uint32_t a) {
  uint64_t v; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a)); return v;
}
__device__ __forceinline__ float4 ld_s128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void st_s64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.b64 [%0], %1;" :: "r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void mb_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(a) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(bytes) : "memory");
}
// ST_WAIT2 (experiment): 0 = try_wait with a suspend-time hint (default), 1 = try_wait without
// a hint, 2 = test_wait spin
#ifndef ST_WAIT2
#define ST_WAIT2 0
#endif
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  do {
#if ST_WAIT2 == 2
    asm volatile("{\n\t.reg .pred q;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
#elif ST_WAIT2 == 1
    asm volatile("{\n\t.reg .pred q;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
#else
    asm volatile("{\n\t.reg .pred q;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, 0x989680;\n\t"
                 "selp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
#endif
  } while (!ok);
}
__device__ __forceinline__ void tma_load_3d_s(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                              int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async8_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}

template <int R, int TK, bool WAVE, int OY_>
struct Geom2 {
  static constexpr int VY = 2;                     // rows per warp
  static constexpr int GW = 64;
  static constexpr int QN = 2 * R + 1;
  static constexpr int OY = OY_;
  static constexpr int GH = OY + 2 * (TK - 1) * R; // level-0 rows
  static constexpr int rows(int l) { return GH - 2 * l * R; }
  static constexpr int warps(int l) { return rows(l) / VY; }
  static constexpr int wbase(int l) { return l == 0 ? 0 : wbase(l - 1) + warps(l - 1); }
  static constexpr int NCW = wbase(TK);            // consumer warps over all levels
  static constexpr int NPROD = WAVE ? 2 : 1;       // producer warps: u^n ring (+ E rings, wave)
  static constexpr int NTHREADS = 32 * (NCW + NPROD);
  static constexpr int RXB = (R + 3) & ~3;
  static constexpr int HX0 = Halo<R, TK>::hx(0);   // level-0 x halo (even)
  static constexpr int XS = HX0 % 4;               // keep the TMA box start 16-B aligned
  static constexpr int BW = GW + 2 * RXB + (XS ? 8 : 0);
  static constexpr int BH = GH + 2 * R;
  static constexpr int BCOL = RXB + XS;
  static constexpr int OX = GW - 2 * HX0;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
#ifndef ST_DL2
#define ST_DL2 2
#endif
  static constexpr int DL = R + ST_DL2;            // level-ring depth (planes); >= R + 1 needed
  static constexpr int LVL_BYTES = GW * (GH + 2 * R) * 4;   // one plane + R pad rows each side
#ifndef ST_DE2
#define ST_DE2 0        // 0: as deep as shared memory allows (below)
#endif
#ifndef ST_ROT2
#define ST_ROT2 0
#endif
  // producer-streamed boxes (wave): level 0 gets u^{n-1} and the medium of its plane (GH rows),
  // level 1 gets u^n and the medium of its plane (OY rows); DE entries per ring.
  static constexpr int XSE = HX0 % 4;              // keep the field box start 16-B aligned
  static constexpr int EBW = GW + (XSE ? 4 : 0);   // field box width (floats)
  // field part first (padded to 128 B: TMA destinations are 128-B aligned), then the medium
  static constexpr int E0_FIELD = (EBW * GH * 4 + 127) / 128 * 128, E0_BYTES = E0_FIELD + 128 * GH * 4;
  static constexpr int E1_FIELD = (EBW * OY * 4 + 127) / 128 * 128, E1_BYTES = E1_FIELD + 128 * OY * 4;
  // E-ring depth: as deep as the shared memory left after the level rings and a u^n ring of
  // R + 3 slots allows (2..8); measured: deeper E rings hide the DRAM latency of the medium.
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int DE_FIT = (SMEM_MAX - 2048 - (TK - 1) * DL * LVL_BYTES - (R + 3) * SLOT_BYTES) /
                                (E0_BYTES + E1_BYTES);
  static constexpr int DE = ST_DE2 ? ST_DE2 : (DE_FIT < 2 ? 2 : DE_FIT > 8 ? 8 : DE_FIT);
  static constexpr int BAR_BYTES = 2048;   // full[64] | empty[64] | lfull | lempty | E0 f/e | E1 f/e
  static constexpr int EBAR_OFF = 1792;
  static constexpr int LRING_OFF = BAR_BYTES;
  static constexpr int E0_OFF = LRING_OFF + (TK - 1) * DL * LVL_BYTES;
  static constexpr int E1_OFF = E0_OFF + (WAVE ? DE * E0_BYTES : 0);
  static constexpr int FIXED_BYTES = E1_OFF + (WAVE ? DE * E1_BYTES : 0);
  static_assert(1024 + 16 * (TK - 1) * DL <= EBAR_OFF && EBAR_OFF + 32 * DE <= BAR_BYTES, "barrier area");
  static_assert(TK >= 2 && (!WAVE || TK == 2), "time-tiled kernel: wave TK = 2, heat TK >= 2");
  static_assert(OY % 2 == 0 && NCW + NPROD <= 32, "warp budget");
  static_assert(OX > 0, "tile too small for this radius / depth");
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
  static_assert(FIXED_BYTES % 128 == 0, "TMA ring alignment");
};

// x/y/z accumulation of two rows (canonical order, include/stencil.h).  cb: shared address of
// (my first row, my pair) in the centre plane; PB: plane row pitch in bytes; q: z-queue whose
// centre is q[R].
template <int R, int PB>
__device__ __forceinline__ void accum2(uint64_t (&acc)[2], const uint64_t (&q)[2 * R + 1][2],
                                       uint32_t cb, const SweepParams& p, const int CI) {
  constexpr int RX2 = (R + 1) & ~1;
  constexpr int QN = 2 * R + 1;
  const uint64_t K0 = splat(p.K0);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint32_t rb = cb + j * PB;
    const uint64_t c = q[CI][j];
    uint64_t A[RX2 + 1];
#pragma unroll
    for (int m = -RX2 / 2; m <= RX2 / 2; ++m) {
      A[m + RX2 / 2] = (m == 0) ? c : ld_s64r(rb + 8 * m);
    }
    uint64_t a = f2mul(K0, c);
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      uint64_t sx;
      if ((k & 1) == 0) {
        sx = f2add(A[RX2 / 2 - k / 2], A[RX2 / 2 + k / 2]);
      } else {   // odd offset: element sums taken from neighbouring aligned pairs
        const uint64_t Lm = A[RX2 / 2 - (k + 1) / 2], L0 = A[RX2 / 2 - (k - 1) / 2];
        const uint64_t R0 = A[RX2 / 2 + (k - 1) / 2], Rp = A[RX2 / 2 + (k + 1) / 2];
        sx = pack2(fadd_ftz(hi_of(Lm), hi_of(R0)), fadd_ftz(lo_of(L0), lo_of(Rp)));
      }
      a = f2fma(splat(p.W[0][k]), sx, a);
      const uint64_t yl = (j - k >= 0) ? q[CI][(j - k) >= 0 ? (j - k) : 0] : ld_s64r(rb - k * PB);
      const uint64_t yr = (j + k < 2) ? q[CI][(j + k) < 2 ? (j + k) : 0] : ld_s64r(rb + k * PB);
      a = f2fma(splat(p.W[1][k]), f2add(yl, yr), a);
      a = f2fma(splat(p.W[2][k]), f2add(q[md<QN>(CI - k)][j], q[md<QN>(CI + k)][j]), a);
    }
    acc[j] = a;
  }
}

// One consumer warp of level L (group L): the whole z stream of the CTA's chunk.
template <int L, int R, int TK, bool WAVE, int OY, bool SAVE>
__device__ __forceinline__ void level_warp(const SweepParams& p, const int nslot, const uint32_t sbase,
                                           const int warp, const int lane, const int tx0,
                                           const int ty0, const int zb, const int ze) {
  using G = Geom2<R, TK, WAVE, OY>;
  constexpr int QN = G::QN, GW = G::GW, BW = G::BW, DL = G::DL, DE = G::DE, GH = G::GH;
  constexpr int HX0 = G::HX0, HY0 = (TK - 1) * R;
  constexpr int SLOT = G::SLOT_BYTES, LVL = G::LVL_BYTES;
  constexpr int EB = (L == 0) ? G::E0_BYTES : G::E1_BYTES;            // E-ring entry
  constexpr int EFIELD = (L == 0) ? G::E0_FIELD : G::E1_FIELD;        // medium part offset
  constexpr int PB = (L == 0) ? BW * 4 : GW * 4;   // input-plane row pitch (bytes)
  const int wl = warp - G::wbase(L);
  const int r0 = L * R + 2 * wl;                    // region row of my first row
  const int gx = tx0 - HX0, gy = ty0 - HY0;
  const int x0 = gx + 2 * lane;
  const bool xin0 = (x0 >= 0) && (x0 < p.nx);
  const bool xin1 = (x0 + 1 >= 0) && (x0 + 1 < p.nx);
  const uint64_t xmask = (xin0 ? 0xffffffffull : 0ull) | (xin1 ? 0xffffffff00000000ull : 0ull);
  const int y0 = gy + r0;
  const bool yin0 = (y0 >= 0) && (y0 < p.ny), yin1 = (y0 + 1 >= 0) && (y0 + 1 < p.ny);
  const uint64_t m0 = yin0 ? xmask : 0ull, m1 = yin1 ? xmask : 0ull;
  const bool lane_out = (lane >= HX0 / 2) && (lane < 32 - HX0 / 2);   // output-tile lanes
  const bool row0_out = r0 >= HY0 && r0 < GH - HY0, row1_out = r0 + 1 >= HY0 && r0 + 1 < GH - HY0;
  // last level: the warp's output columns [tx0, tx0 + OX) and both rows are interior
  const bool whole = (tx0 + G::OX <= p.nx) && yin0 && yin1;
  const int p_first = zb - TK * R;
  const int n_arr = (ze - zb) + 2 * TK * R;
  // level L at step a computes plane p_first + a - (L+1)R; active on [a_lo, a_hi)
  const int q_lo = max(zb - (TK - 1 - L) * R, p.gz_lo), q_hi = min(ze + (TK - 1 - L) * R, p.gz_hi);
  const int a_lo = q_lo - p_first + (L + 1) * R, a_hi = q_hi - p_first + (L + 1) * R;

  // rare events (warp-uniform)
  bool wsrc = false, wrec = false;
  if (q_lo < q_hi) {
    if (yin0) wsrc |= row_has_entry(p.src_begin, p.src, q_lo, q_hi, y0, gx, gx + 64);
    if (yin1) wsrc |= row_has_entry(p.src_begin, p.src, q_lo, q_hi, y0 + 1, gx, gx + 64);
  }
  if (yin0 && row0_out) wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0, tx0, tx0 + G::OX);
  if (yin1 && row1_out) wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + 1, tx0, tx0 + G::OX);
  wsrc = __any_sync(0xffffffffu, wsrc);
  wrec = __any_sync(0xffffffffu, wrec);

  // shared-window addresses
  const uint32_t b_full = sbase, b_empty = sbase + 512;
  const uint32_t b_lf = sbase + 1024, b_le = sbase + 1024 + 8 * (TK - 1) * DL;
  const uint32_t lf_in = b_lf + 8 * ((L > 0 ? L - 1 : 0) * DL), le_in = b_le + 8 * ((L > 0 ? L - 1 : 0) * DL);
  const uint32_t lf_out = b_lf + 8 * ((L < TK - 1 ? L : 0) * DL), le_out = b_le + 8 * ((L < TK - 1 ? L : 0) * DL);
  const uint32_t ring_in = (L == 0) ? sbase + G::FIXED_BYTES
                                    : sbase + G::LRING_OFF + (L > 0 ? L - 1 : 0) * DL * LVL;
  const uint32_t ring_out = sbase + G::LRING_OFF + (L < TK - 1 ? L : 0) * DL * LVL;
  const uint32_t my_in = (L == 0) ? ((r0 + R) * BW + G::BCOL + 2 * lane) * 4 : ((r0 + R) * GW + 2 * lane) * 4;
  const uint32_t my_out = ((r0 + R) * GW + 2 * lane) * 4;
  // E ring (wave): level 0 reads ring E0 (rows = region rows), level 1 ring E1 (rows from R)
  const uint32_t e_base = sbase + ((L == 0) ? G::E0_OFF : G::E1_OFF);
  const uint32_t e_full = sbase + G::EBAR_OFF + ((L == 0) ? 0 : 16 * DE), e_empty = e_full + 8 * DE;
  const int er = r0 - L * R;                         // my first row inside the E box
  const uint32_t my_ef = (er * G::EBW + G::XSE + 2 * lane) * 4;      // field pair, row er
  const uint32_t my_ea = EFIELD + (er * 128 + 4 * lane) * 4;          // medium float4, row er
  const long long plane = p.plane;
  const int X = p.X;
  uint64_t q[QN][2];
#pragma unroll
  for (int i = 0; i < QN; ++i) q[i][0] = q[i][1] = 0ull;

  // ring counters
  int in_slot = 0;  uint32_t in_ph = 0;            // input slot of step a
  int c_slot = (L == 0) ? (R % nslot) : 0;         // centre slot (TMA: arrival a-R; ring: step a-R)
  int out_slot = 0; uint32_t out_ph = 0;           // output ring slot of step a
  int e_slot = 0; uint32_t e_ph = 0;               // E-ring entry of step a
  const uint64_t DT = splat(p.dt);
  const bool wr_prev = WAVE || p.write_prev;
  const long long obase = (long long)(p_first - TK * R) * plane + (long long)y0 * X + x0;

  // ST_ROT2 = 1: the z-queue is rotated by register moves after each step (code = one step
  // body); 0: the loop is unrolled by the queue length and the queue indexed modulo QN.
  constexpr int UNR = ST_ROT2 ? 1 : QN;
#pragma unroll 1
  for (int base = 0; base < n_arr; base += UNR) {
#pragma unroll
  for (int uu = 0; uu < UNR; ++uu) {
    const int a = base + uu;
    if (a >= n_arr) break;
    const int iN = ST_ROT2 ? QN - 1 : uu;            // queue index of the newest plane
    const int iC = ST_ROT2 ? R : md<QN>(uu - R);     // queue index of the centre plane
    // ---- input plane of step a into the queue ----------------------------------------------
    if (L == 0) {
      mb_wait(b_full + 8 * in_slot, in_ph);
      const uint32_t s = ring_in + in_slot * SLOT + my_in;
      q[iN][0] = ld_s64<0>(s);
      q[iN][1] = ld_s64<PB>(s);
      // never a centre plane: release now, once this lane's loads from the slot have returned
      if (a < R) mb_arrive(b_empty + 8 * in_slot + (zero_after(q[iN][0], p.zero) | zero_after(q[iN][1], p.zero)));
      if (++in_slot == nslot) { in_slot = 0; in_ph ^= 1u; }
    } else {
      mb_wait(lf_in + 8 * in_slot, in_ph);
      const uint32_t s = ring_in + in_slot * LVL + my_in;
      q[iN][0] = ld_s64<0>(s);
      q[iN][1] = ld_s64<PB>(s);
      if (++in_slot == DL) { in_slot = 0; in_ph ^= 1u; }
    }
    // ---- this step's E entry (wave) ----------------------------------------------------------
    if (WAVE) mb_wait(e_full + 8 * e_slot, e_ph);

    // ---- level L at plane p_first + a - (L+1)R ----------------------------------------------
    uint64_t o0 = 0ull, o1 = 0ull;
    const bool centre = (L == 0) ? (a >= 2 * R) : (a >= R);
    if (centre) {
      if (a >= a_lo && a < a_hi) {
        const int qp = p_first + a - (L + 1) * R;
        const uint32_t cb = ring_in + c_slot * ((L == 0) ? SLOT : LVL) + my_in;
        uint64_t acc[2];
        accum2<R, PB>(acc, q, cb, p, iC);
        if (wsrc) {
          if (yin0) acc[0] = add_sources_row(acc[0], p, qp, y0, x0, p.wl_step + L);
          if (yin1) acc[1] = add_sources_row(acc[1], p, qp, y0 + 1, x0, p.wl_step + L);
        }
        const uint64_t c0 = q[iC][0], c1 = q[iC][1];
        if (WAVE) {
          const uint32_t e = e_base + e_slot * EB;
          const uint64_t p0 = ld_s64r(e + my_ef), p1 = ld_s64r(e + my_ef + G::EBW * 4);
          const float4 a0 = ld_s128(e + my_ea), a1 = ld_s128(e + my_ea + 128 * 4);
          o0 = f2fma(pack2(a0.z, a0.w), acc[0], f2fma(pack2(a0.x, a0.y), f2sub(p0, c0), c0));
          o1 = f2fma(pack2(a1.z, a1.w), acc[1], f2fma(pack2(a1.x, a1.y), f2sub(p1, c1), c1));
        } else {
          o0 = f2fma(DT, acc[0], c0);
          o1 = f2fma(DT, acc[1], c1);
        }
        o0 &= m0; o1 &= m1;
        if (L == TK - 1) {
          // u^{n+TK} and u^{n+TK-1} on the output tile (every row of the last group is an
          // output row; the active range is exactly the output planes)
          if (whole) {                 // warp-uniform: both rows and all columns interior
            if (lane_out) {
              const long long off = obase + (long long)a * plane;
              sts64(p.outC + off, o0); sts64(p.outC + off + X, o1);
              if (wr_prev) { sts64(p.outP + off, c0); sts64(p.outP + off + X, c1); }
              if (SAVE) { sts64(p.outS + off, o0); sts64(p.outS + off + X, o1); }
            }
          } else if (lane_out && xin0) {
            const long long off = obase + (long long)a * plane;
            float* oc = p.outC + off;
            float* op = p.outP + off;
            if (xin1) {
              if (yin0) { sts64(oc, o0); if (wr_prev) sts64(op, c0); }
              if (yin1) { sts64(oc + X, o1); if (wr_prev) sts64(op + X, c1); }
            } else {
              if (yin0) { oc[0] = lo_of(o0); if (wr_prev) op[0] = lo_of(c0); }
              if (yin1) { oc[X] = lo_of(o1); if (wr_prev) op[X] = lo_of(c1); }
            }
            if (SAVE) {   // snapshot of u^{n+TK}
              float* os = p.outS + off;
              if (xin1) { if (yin0) sts64(os, o0); if (yin1) sts64(os + X, o1); }
              else { if (yin0) os[0] = lo_of(o0); if (yin1) os[X] = lo_of(o1); }
            }
          }
        }
        if (wrec && qp >= zb && qp < ze && lane_out) {
          if (yin0 && row0_out) sample_receivers_row(o0, p, qp, y0, x0, p.tr_step + L);
          if (yin1 && row1_out) sample_receivers_row(o1, p, qp, y0 + 1, x0, p.tr_step + L);
        }
      }
      // release the centre plane
      if (L == 0) {
        mb_arrive(b_empty + 8 * c_slot);
        if (++c_slot == nslot) c_slot = 0;
      } else {
        mb_arrive(le_in + 8 * c_slot);
        if (++c_slot == DL) c_slot = 0;
      }
    }
    if (WAVE) {
      mb_arrive(e_empty + 8 * e_slot);
      if (++e_slot == DE) { e_slot = 0; e_ph ^= 1u; }
    }

    // ---- publish level L's plane into its ring (levels below the last) -----------------------
    if (L < TK - 1) {
      if (a >= DL) mb_wait(le_out + 8 * out_slot, out_ph ^ 1u);
      const uint32_t d = ring_out + out_slot * LVL + my_out;
      st_s64(d, o0);
      st_s64(d + GW * 4, o1);
      mb_arrive(lf_out + 8 * out_slot);
      if (++out_slot == DL) { out_slot = 0; out_ph ^= 1u; }
    }

    // ---- rotate the z-queue -------------------------------------------------------------------
    if (ST_ROT2) {
#pragma unroll
      for (int i = 0; i + 1 < QN; ++i) { q[i][0] = q[i + 1][0]; q[i][1] = q[i + 1][1]; }
    }
  }
  }
}

template <int L, int R, int TK, bool WAVE, int OY, bool SAVE>
__device__ __forceinline__ void dispatch_level(int l, const SweepParams& p, int nslot, uint32_t sbase,
                                               int warp, int lane, int tx0, int ty0, int zb, int ze) {
  if (l == L) {
    level_warp<L, R, TK, WAVE, OY, SAVE>(p, nslot, sbase, warp, lane, tx0, ty0, zb, ze);
  } else if constexpr (L + 1 < TK) {
    dispatch_level<L + 1, R, TK, WAVE, OY, SAVE>(l, p, nslot, sbase, warp, lane, tx0, ty0, zb, ze);
  }
}

// SAVE: the pass also stores u^{n+TK} into the snapshot field p.outS (separate instance).
template <int R, int TK, bool WAVE, int OY, bool SAVE>
#ifndef ST_MINB2
#define ST_MINB2 1      // experiment: resident CTAs per SM the register allocation must allow
#endif
__global__ void __launch_bounds__(Geom2<R, TK, WAVE, OY>::NTHREADS, ST_MINB2)
sweep2_kernel(const __grid_constant__ KernelMaps maps, const __grid_constant__ SweepParams p,
              const int nslot) {
  using G = Geom2<R, TK, WAVE, OY>;
  constexpr int NCW = G::NCW, DL = G::DL, DE = G::DE;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * G::OX, ty0 = blockIdx.y * G::OY;   // output tile origin
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mb_init(sbase + 8 * i, 1);                          // full: producer's expect_tx
      mb_init(sbase + 512 + 8 * i, 32 * G::warps(0));     // empty: level-0 lanes
    }
    for (int l = 0; l + 1 < TK; ++l)
      for (int i = 0; i < DL; ++i) {
        mb_init(sbase + 1024 + 8 * (l * DL + i), 32 * G::warps(l));                         // writers
        mb_init(sbase + 1024 + 8 * ((TK - 1) * DL + l * DL + i), 32 * G::warps(l + 1));     // readers
      }
    if (WAVE)
      for (int i = 0; i < DE; ++i) {
        mb_init(sbase + G::EBAR_OFF + 8 * i, 1);                        // E0 full (expect_tx)
        mb_init(sbase + G::EBAR_OFF + 8 * (DE + i), 32 * G::warps(0));  // E0 empty
        mb_init(sbase + G::EBAR_OFF + 8 * (2 * DE + i), 1);             // E1 full
        mb_init(sbase + G::EBAR_OFF + 8 * (3 * DE + i), 32 * G::warps(1));
      }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_prologue_done();

  if (warp >= NCW) {
    // ------------------------------------------------------------------ producer warp
    // warp NCW streams the u^n ring, warp NCW+1 (wave) the E rings: separate warps, so the two
    // streams run ahead of their consumers independently (a sleeping try_wait of one stream
    // never holds the other back; each is bounded by its own ring depth).
    const int p_first = zb - TK * R, n_arr = (ze - zb) + 2 * TK * R;
    const int gx = tx0 - G::HX0, gy = ty0 - (TK - 1) * R;
    if (warp == NCW && lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&maps.u)) : "memory");
      const uint32_t ring = sbase + G::FIXED_BYTES;
      int slot = 0;
      uint32_t ph = 0;
      for (int a = 0; a < n_arr; ++a) {
        if (a >= nslot) mb_wait(sbase + 512 + 8 * slot, ph ^ 1u);
        mb_expect_tx(sbase + 8 * slot, (uint32_t)(G::BW * G::BH * 4));
        tma_load_3d_s(ring + slot * G::SLOT_BYTES, &maps.u, sbase + 8 * slot, gx - G::BCOL, gy - R,
                      p_first + a - p.zv_lo);
        if (++slot == nslot) { slot = 0; ph ^= 1u; }
      }
    } else if (WAVE && warp == NCW + 1 && lane == 0) {
      const uint32_t ebar = sbase + G::EBAR_OFF;
      int es = 0;
      uint32_t eph = 0;
      for (int a = 0; a < n_arr; ++a) {
        // level 0 plane s = p_first + a - R (rows gy..), level 1 plane s - R (rows gy + R..)
        const int zs = p_first + a - R - p.zv_lo;
        if (a >= DE) {
          mb_wait(ebar + 8 * (DE + es), eph ^ 1u);
          mb_wait(ebar + 8 * (3 * DE + es), eph ^ 1u);
        }
        const uint32_t f0 = ebar + 8 * es, f1 = ebar + 8 * (2 * DE + es);
        const uint32_t d0 = sbase + G::E0_OFF + es * G::E0_BYTES, d1 = sbase + G::E1_OFF + es * G::E1_BYTES;
        mb_expect_tx(f0, (uint32_t)((G::EBW + 128) * G::GH * 4));
        tma_load_3d_s(d0, &maps.p0, f0, gx - G::XSE, gy, zs);
        tma_load_3d_s(d0 + G::E0_FIELD, &maps.a0, f0, 2 * gx, gy, zs);
        mb_expect_tx(f1, (uint32_t)((G::EBW + 128) * G::OY * 4));
        tma_load_3d_s(d1, &maps.u1, f1, gx - G::XSE, gy + R, zs - R);
        tma_load_3d_s(d1 + G::E1_FIELD, &maps.a1, f1, 2 * gx, gy + R, zs - R);
        if (++es == DE) { es = 0; eph ^= 1u; }
      }
    }
    return;
  }
  int l = 0;
#pragma unroll
  for (int m = 1; m < TK; ++m) l += (warp >= G::wbase(m)) ? 1 : 0;
  dispatch_level<0, R, TK, WAVE, OY, SAVE>(l, p, nslot, sbase, warp, lane, tx0, ty0, zb, ze);
}

}  // namespace st
