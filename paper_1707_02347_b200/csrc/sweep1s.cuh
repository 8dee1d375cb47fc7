// sweep1s.cuh -- untiled (T = 1) 3-D sweep with a STATIC ring: the TMA ring has exactly QN = 2r+1
// slots, so the slot of every arrival, the z-queue index of every plane and the mbarrier of every
// slot are compile-time constants of the QN-fold unrolled step body.
//
// Same schedule and arithmetic as sweep1_kernel (sweep1.cuh: warp-specialised, one TMA producer
// warp, consumers with a register z-queue and a column pair per lane, packed fp32x2, canonical
// per-point order of include/stencil.h), restructured for issue efficiency at high order
// (DESIGN.md §6 G1s):
//   * arrival a lands in ring slot a mod QN and queue entry a mod QN; in unrolled position uu of
//     block b (a = b*QN + uu) both are uu, the centre plane (a - r) is entry/slot (uu - r) mod QN
//     and the full-barrier parity is b & 1 -- no per-step slot arithmetic, no per-step address
//     computation (every shared-memory access is base register + immediate);
//   * block 0 (the r-plane warm-up below the chunk, which only loads) is peeled, so the steady
//     blocks carry no warm-up conditions;
//   * the ring depth QN leaves r planes of TMA prefetch beyond the r+1 planes in use (r >= 5).
// Built for the 3-D wave and heat at r = 5, 6, 8 (build.py _static_ring: there QN slots plus the
// cp.async staging fit in shared memory and it measured faster); other shapes keep sweep1_kernel.
#pragma once
#include "sweep1.cuh"
#include "sweep2.cuh"   // 32-bit shared-window TMA helper

namespace st {

#ifndef ST_S1S_TMAE
#define ST_S1S_TMAE 1   // 1: u^{n-1} and the medium arrive by TMA (second producer warp, E ring);
                        // 0: per-warp cp.async staging (round-1 design, for A/B builds)
#endif

template <int R, int NCW, int VY, bool WAVE>
struct Geom1S {
  using B = Geom1<R, 3, NCW, VY>;
  static constexpr int QN = 2 * R + 1;
  static constexpr int NS = QN;                              // ring slots
  static constexpr int SLOT_BYTES = B::SLOT_BYTES;
  static constexpr int STAGE_F = B::STAGE_F;
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int BAR_BYTES = 1024;
  static constexpr bool TMAE = WAVE && ST_S1S_TMAE;
  // TMA E ring (TMAE): per output plane, the tile's u^{n-1} box (64 x OY), its c box and its a
  // box (planar medium, 64 x OY each); the a box is loaded only where the tile's plane holds a
  // point with a != -1 (damping; SweepParams::aflag) -- elsewhere a is the constant -1 and the
  // sweep moves 16 instead of 20 B/update; DE entries, as many as shared memory allows (<= 8)
  static constexpr int OY = NCW * VY;
  static constexpr int E_FIELD = (64 * OY * 4 + 127) / 128 * 128;
  static constexpr int E_BYTES = 3 * E_FIELD;
  static constexpr int DE_FIT = (SMEM_MAX - BAR_BYTES - NS * SLOT_BYTES) / E_BYTES;
  static constexpr int DE = DE_FIT > 8 ? 8 : DE_FIT;
  static constexpr int stage_bytes(int pd) { return NCW * (pd + 1) * STAGE_F * 4; }
  static constexpr bool fits(int pd) {
    return BAR_BYTES + NS * SLOT_BYTES + (WAVE && !TMAE ? stage_bytes(pd) : 0) <= SMEM_MAX;
  }
  static constexpr int PD = fits(4) ? 4 : 3;                 // cp.async staging distance (planes)
  static constexpr bool OK = TMAE ? DE >= 2 : fits(PD);
  static constexpr int FIXED_BYTES = BAR_BYTES + (TMAE ? DE * E_BYTES : WAVE ? stage_bytes(PD) : 0);
  static constexpr int NPROD = TMAE ? 2 : 1;                 // producer warps
  static constexpr int NTHREADS = 32 * (NCW + NPROD);
  static_assert(!TMAE || (FIXED_BYTES % 128 == 0), "TMA ring alignment");
};

// MODE: 0 plain, 1 snapshot store (SAVE), 2 fused halo push (PUSH), as sweep1_kernel.
template <int R, bool WAVE, int NCW, int VY, int MODE, bool ISO = false>
__global__ void __launch_bounds__(Geom1S<R, NCW, VY, WAVE>::NTHREADS, 1)
sweep1s_kernel(const __grid_constant__ KernelMaps maps, const __grid_constant__ SweepParams p,
               const int nslot_unused) {
  const CUtensorMap& tmapC = maps.u;
  constexpr bool SAVE = MODE == 1, PUSH = MODE == 2;
  using G = Geom1<R, 3, NCW, VY>;
  using S = Geom1S<R, NCW, VY, WAVE>;
  static_assert(S::OK, "static ring does not fit in shared memory");
  constexpr int QN = S::QN, NS = S::NS, BW = G::BW, RXB = G::RXB;
  constexpr int SLOT_F = S::SLOT_BYTES / 4;
  constexpr int PD = S::PD, STAGE_F = S::STAGE_F;
  constexpr bool TMAE = S::TMAE;
  constexpr int DE = S::DE, EB = S::E_BYTES;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NS;
  uint64_t* efull = full + 2 * NS;                // E ring (TMAE)
  uint64_t* eempty = efull + 8;
  volatile uint32_t* eflag = reinterpret_cast<volatile uint32_t*>(eempty + 8);   // per E entry: a == -1
  float* stage0 = reinterpret_cast<float*>(smem + S::BAR_BYTES);
  float* ring = reinterpret_cast<float*>(smem + S::FIXED_BYTES);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * G::OX, ty0 = blockIdx.y * G::OY;
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;
  const int p_first = zb - R;
  const int n_arr = (ze - zb) + 2 * R;          // >= QN

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 32 * NCW);
    }
    if (TMAE)
      for (int i = 0; i < DE; ++i) {
        mbar_init(&efull[i], 1);
        mbar_init(&eempty[i], 32 * NCW);
      }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_prologue_done();

  if (TMAE && warp == NCW + 1) {
    // ------------------------------------------------- producer warp 2: u^{n-1} + medium per plane
    if (lane == 0) {
      int es = 0;
      uint32_t eph = 0;
      const uint32_t ebase = smem_u32(smem + S::BAR_BYTES);
      const long long fl_stride = (long long)p.fl_nty * p.fl_ntx;
      const unsigned char* fl = p.aflag + zb * fl_stride + (long long)blockIdx.y * p.fl_ntx + blockIdx.x;
      uint32_t f_next = ld_flag(fl);
      for (int s = zb; s < ze; ++s) {
        const uint32_t f = f_next;                       // 1: a == -1 on this tile's plane s
        fl += fl_stride;
        if (s + 1 < ze) f_next = ld_flag(fl);            // in flight across the wait below
        if (s - zb >= DE) mbar_wait(&eempty[es], eph ^ 1u);
        eflag[es] = f;                                   // released to the consumers by the arrive
        mbar_expect_tx(&efull[es], (uint32_t)((f ? 2 : 3) * 64 * S::OY * 4));   // OOB zero-filled
        tma_load_3d_s(ebase + es * EB, &maps.p0, smem_u32(&efull[es]), tx0, ty0, s - p.zv_lo);
        tma_load_3d_s(ebase + es * EB + S::E_FIELD, &maps.a0, smem_u32(&efull[es]), tx0, ty0, s - p.zv_lo);
        if (!f)
          tma_load_3d_s(ebase + es * EB + 2 * S::E_FIELD, &maps.a1, smem_u32(&efull[es]), tx0, ty0, s - p.zv_lo);
        if (++es == DE) { es = 0; eph ^= 1u; }
      }
    }
    return;
  }
  if (warp == NCW) {
    // ------------------------------------------------------------------ producer warp
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapC)) : "memory");
      int slot = 0;
      uint32_t ph = 0;
      bool lo_done = false, hi_done = false;
      for (int a = 0; a < n_arr; ++a) {
        if (a >= NS) mbar_wait(&empty[slot], ph ^ 1u);
        if (PUSH) wait_ghost(p, p_first + a, lo_done, hi_done);   // neighbour's push landed
        mbar_expect_tx(&full[slot], (uint32_t)(BW * G::BH * 4));
        tma_load_3d(ring + (size_t)slot * SLOT_F, &tmapC, &full[slot], tx0 - RXB, ty0 - R,
                    p_first + a - p.zv_lo);
        if (++slot == NS) { slot = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  const int x0 = tx0 + 2 * lane;
  const int y0 = ty0 + warp * VY;
  const bool xin0 = x0 < p.nx, xin1 = x0 + 1 < p.nx;
  const uint64_t xmask = (xin0 ? 0xffffffffull : 0ull) | (xin1 ? 0xffffffff00000000ull : 0ull);
  bool yin[VY];
  uint64_t mask[VY];
  bool any_row = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    yin[j] = y0 + j < p.ny;
    mask[j] = yin[j] ? xmask : 0ull;
    any_row |= yin[j];
  }
  const bool act = any_row && xin0;
  const bool whole = (tx0 + 64 <= p.nx) && (y0 + VY <= p.ny);   // warp-uniform: plain stores
  // fused halo push (CTA-uniform): this chunk produces planes of the lo / hi band
  const bool push_lo = PUSH && p.push_lo != nullptr && zb < p.band_lo;
  const bool push_hi = PUSH && p.push_hi != nullptr && ze > p.band_hi;
  const bool push_any = push_lo || push_hi;
  const float* rcol = ring + (warp * VY + R) * BW + 2 * lane + RXB;   // my pair, slot 0
  const uint64_t DT = splat(p.dt);
  bool wsrc = false, wrec = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    if (yin[j]) {
      wsrc |= row_has_entry(p.src_begin, p.src, zb, ze, y0 + j, tx0, tx0 + 64);
      wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + j, tx0, tx0 + 64);
    }
  }

  const long long plane = p.plane;
  const int X = p.X, X2 = p.X >> 1;
  float* stage = stage0 + (size_t)warp * (PD + 1) * STAGE_F;
  const float* gP = p.P + (long long)zb * plane + (long long)y0 * X + x0;
  const float4* gA = p.ac + (long long)zb * (plane >> 1) + (long long)y0 * X2 + (x0 >> 1);
  float* out = p.outP + (long long)zb * plane + (long long)y0 * X + x0;
  float* outs = SAVE ? p.outS + (long long)zb * plane + (long long)y0 * X + x0 : nullptr;
  int q_iss = zb;
  float* e_iss = stage;                          // staging entry of plane q_iss
  const float* e_use = stage;                    // staging entry of the plane being computed
  float* const stage_end = stage + (PD + 1) * STAGE_F;
  auto stage_next = [&]() {
    if (q_iss < ze && act) {
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (yin[j]) {
          cp_async8(e_iss + j * 64 + 2 * lane, gP + j * X);
          cp_async16(e_iss + VY * 64 + j * 128 + 4 * lane, gA + j * X2);
        }
      }
    }
    cp_async_commit();
    gP += plane; gA += plane >> 1; ++q_iss;
    e_iss += STAGE_F;
    if (e_iss == stage_end) e_iss = stage;
  };
  if (WAVE && !TMAE) {
#pragma unroll 1
    for (int i = 0; i < PD; ++i) stage_next();
  }
  // E ring (TMAE): my u^{n-1} pair and medium float4 of row j inside an entry
  const float* e_slot = reinterpret_cast<const float*>(smem + S::BAR_BYTES);
  const int e_pv = (warp * VY) * 64 + 2 * lane;
  const int e_c = S::E_FIELD / 4 + e_pv, e_a = 2 * (S::E_FIELD / 4) + e_pv;
  const uint64_t NEG1 = splat(-1.0f);
  int es = 0;
  uint32_t eph = 0;

  uint64_t qn[QN][VY];
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) qn[i][j] = 0ull;

  // one output plane: centre = queue entry / ring slot CS (compile-time after unrolling)
  auto compute = [&](const int CS, const int s) {
    if (WAVE && !TMAE) stage_next();              // plane s + PD
    uint64_t acc[VY];
    accumulate<R, R, QN, VY, 3, BW, ISO>(acc, qn, rcol + CS * SLOT_F, p, CS);
    if (wsrc) {
#pragma unroll
      for (int j = 0; j < VY; ++j)
        if (yin[j]) acc[j] = add_sources_row(acc[j], p, s, y0 + j, x0, p.wl_step);
    }
    uint64_t o[VY];
    if (TMAE) {
      // (loading the E entry before the Laplacian measured no faster: C5 304.0 vs 306.6 GPts/s)
      mbar_wait(&efull[es], eph);
      const float* e = e_slot + es * (EB / 4);
      const uint32_t aneg = eflag[es];            // a == -1 on this plane of the tile: no a box
      uint32_t z = aneg & p.zero;
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        const uint64_t c = qn[CS][j];
        const uint64_t pv = lds64(e + e_pv + j * 64);
        const uint64_t cv = lds64(e + e_c + j * 64);
        uint64_t av = NEG1;
        if (!aneg) av = lds64(e + e_a + j * 64);
        z |= zero_after(pv | cv | av, p.zero);
        o[j] = f2fma(cv, acc[j], f2fma(av, f2sub(pv, c), c)) & mask[j];
      }
      mbar_arrive(&eempty[es] + z);      // release the entry once my loads from it have returned
      if (++es == DE) { es = 0; eph ^= 1u; }
    } else if (WAVE) {
      cp_async_wait<PD>();
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        const uint64_t c = qn[CS][j];
        const uint64_t pv = lds64(e_use + j * 64 + 2 * lane);
        const float4 m4 = *reinterpret_cast<const float4*>(e_use + VY * 64 + j * 128 + 4 * lane);
        o[j] = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c)) & mask[j];
      }
      e_use += STAGE_F;
      if (e_use == stage_end) e_use = stage;
    } else {
#pragma unroll
      for (int j = 0; j < VY; ++j) o[j] = f2fma(DT, acc[j], qn[CS][j]) & mask[j];
    }
    auto put = [&](float* d) {       // whole tile: plain stores; ragged: masked
      if (whole) {
#pragma unroll
        for (int j = 0; j < VY; ++j) sts64(d + j * X, o[j]);
      } else if (act) {
#pragma unroll
        for (int j = 0; j < VY; ++j) {
          if (yin[j]) {
            if (xin1) sts64(d + j * X, o[j]);
            else d[j * X] = lo_of(o[j]);
          }
        }
      }
    };
    put(out);
    if (SAVE) put(outs);
    if (PUSH && push_any) {            // fused halo: band planes also into the neighbour's ghosts
      if (s < p.band_lo) put(p.push_lo + (out - p.outP));
      if (s >= p.band_hi) put(p.push_hi + (out - p.outP));
    }
    if (wrec) {
#pragma unroll
      for (int j = 0; j < VY; ++j)
        if (yin[j]) sample_receivers_row(o[j], p, s, y0 + j, x0, p.tr_step);
    }
    mbar_arrive(&empty[CS]);
    out += plane;
    if (SAVE) outs += plane;
  };

  // ---- block 0: arrivals 0..QN-1 (planes zb-R .. zb+R); only the last one computes (plane zb)
#pragma unroll
  for (int uu = 0; uu < QN; ++uu) {
    mbar_wait(&full[uu], 0u);
#pragma unroll
    for (int j = 0; j < VY; ++j) qn[uu][j] = lds64(rcol + uu * SLOT_F + j * BW);
    if (uu < R) {
      // never a centre plane: release at once, but only after this lane's loads have returned
      // (same reasoning as sweep1_kernel)
      uint32_t z = 0;
#pragma unroll
      for (int j = 0; j < VY; ++j) z |= zero_after(qn[uu][j], p.zero);
      mbar_arrive(&empty[uu] + z);
    }
    if (uu == QN - 1) compute(md<QN>(uu - R), zb);
  }
  // ---- steady blocks: every arrival computes the plane r below it
  uint32_t ph = 1u;
  int s = zb + 1;
#pragma unroll 1
  for (int base = QN; base < n_arr; base += QN) {
#pragma unroll
    for (int uu = 0; uu < QN; ++uu) {
      if (base + uu < n_arr) {
        mbar_wait(&full[uu], ph);
#pragma unroll
        for (int j = 0; j < VY; ++j) qn[uu][j] = lds64(rcol + uu * SLOT_F + j * BW);
        compute(md<QN>(uu - R), s);
        ++s;
      }
    }
    ph ^= 1u;
  }
  if (WAVE && !TMAE) cp_async_wait<0>();
  if (PUSH) signal_peers(p, push_lo, push_hi, 32 * NCW);
}

}  // namespace st
