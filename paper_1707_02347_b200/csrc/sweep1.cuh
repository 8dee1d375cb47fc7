// sweep1.cuh -- untiled (one time level per pass) 2.5-D sweep for sm_100a, warp-specialised.
//
// The T=1 member of the schedule family (Devito's space-only blocking; SURVEY §8
// row a2/a3).  One CTA = one x-y tile of 64 x NCW points streaming z:
//   * warp NCW (producer): one elected lane issues the TMA load of every u^n plane box
//     (tile + radius halo, OOB zero-filled = Dirichlet) into a ring of NSLOT shared-memory slots,
//     waiting on the slot's EMPTY mbarrier before reuse and arming its FULL mbarrier;
//   * warps 0..NCW-1 (consumers): warp w owns row w of the tile, a column PAIR per lane (packed
//     fp32x2 math).  Each keeps its own z-column of 2r+1 planes in registers, reads x/y
//     neighbours from the ring slot of the centre plane, computes u^{n+1} in the canonical order
//     (include/stencil.h), stores it in place over u^{n-1}, and releases the slot (EMPTY arrive).
// Consumers never synchronise with each other, so warps drift within the ring depth and HBM
// latency hides behind the other warps' work; u^{n-1} and the medium (a, c) are staged PD planes
// ahead into per-warp shared memory with cp.async (LDGSTS) and waited for with wait_group, so no
// register ever waits on a fresh load.  The body is unrolled by the queue length only (one row per
// warp) and carries no per-step division, 64-bit index math or table lookups, which keeps the
// loop small (instruction-cache resident) and the issue slots for the stencil arithmetic.
#pragma once
#include "sweep.cuh"

namespace st {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async8(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float4* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

__device__ __forceinline__ void tma_load_3d_e(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                              int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

// Rare paths kept out of the unrolled body (called only by warps whose row holds an event).
static __device__ __noinline__ uint64_t add_sources_row(uint64_t acc, const SweepParams& p, int s, int y,
                                                 int x0, long long wl_step) {
  const int sb = __ldg(p.src_begin + s), se = __ldg(p.src_begin + s + 1);
  for (int i = sb; i < se; ++i) {
    const int4 e = __ldg(p.src + i);
    if (e.y == y && (e.x == x0 || e.x == x0 + 1)) {
      const float w = __ldg(p.wavelet + wl_step * p.wl_stride + e.w);
      acc = (e.x == x0) ? pack2(fadd_ftz(lo_of(acc), w), hi_of(acc))
                        : pack2(lo_of(acc), fadd_ftz(hi_of(acc), w));
    }
  }
  return acc;
}
static __device__ __noinline__ void sample_receivers_row(uint64_t o, const SweepParams& p, int s, int y,
                                                  int x0, int tr_step) {
  const int rb = __ldg(p.rec_begin + s), re = __ldg(p.rec_begin + s + 1);
  for (int i = rb; i < re; ++i) {
    const int4 e = __ldg(p.rec + i);
    if (e.y == y && (e.x == x0 || e.x == x0 + 1))
      p.trace[(long long)tr_step * p.tr_stride + e.w] = (e.x == x0) ? lo_of(o) : hi_of(o);
  }
}

template <int R, int NDIM, int NCW, int VY = 1>
struct Geom1 {
  static constexpr int RZ = (NDIM == 3) ? R : 0;
  static constexpr int QN = 2 * RZ + 1;
  static constexpr int RX2 = (R + 1) & ~1;
  static constexpr int RXB = (R + 3) & ~3;         // box x halo, multiple of 4 floats (16 B)
  static constexpr int GW = 64, GH = NCW * VY;   // VY rows per consumer warp
  static constexpr int BW = GW + 2 * RXB;          // multiple of 8 floats
  static constexpr int BH = GH + 2 * R;
  static constexpr int OX = GW, OY = GH;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
  static constexpr int NTHREADS = 32 * (NCW + 1);
#ifndef ST_PD
#define ST_PD 0          // 0: per-geometry default below
#endif
#ifndef ST_ROT1
#define ST_ROT1 0
#endif
  static constexpr int PD = ST_PD ? ST_PD : 4;     // cp.async staging distance (planes)
  static constexpr int STAGE_F = VY * (64 + 128);  // staged plane rows: u^{n-1} (VY x 64) + {a,c} (VY x 128)
  static constexpr int STAGE_BYTES = NCW * (PD + 1) * STAGE_F * 4;
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
};

#ifndef ST_S1_TMAE
#define ST_S1_TMAE 1    // 3-D wave: u^{n-1} and the medium arrive by TMA (E ring, second producer warp)
#endif
// one flag byte of SweepParams::aflag (read-only for the whole launch)
__device__ __forceinline__ uint32_t ld_flag(const unsigned char* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// E ring of the untiled 3-D wave kernels: per output plane, the tile's u^{n-1} box (64 x OY), its
// c box and -- only where the tile's plane holds a point with a != -1 (SweepParams::aflag) -- its
// a box (planar medium, 64 x OY each), DE entries.  TMA writes into shared memory
// do not use the 128 B/clk/SM LDS crossbar that cp.async staging fills twice.
template <int R, int NDIM, int NCW, int VY, bool WAVE>
struct Geom1E {
  // measured (same box): C3 SO8 332.8 vs 320.6 GPts/s with the E ring; wave SO2 323.6 vs 334.2
  static constexpr bool TMAE = WAVE && NDIM == 3 && R >= 3 && ST_S1_TMAE;
  static constexpr int OY = NCW * VY;
  static constexpr int E_FIELD = (64 * OY * 4 + 127) / 128 * 128;
  static constexpr int E_BYTES = 3 * E_FIELD;
  static constexpr int DE = 4;
  static constexpr int NPROD = TMAE ? 2 : 1;
  static constexpr int NTHREADS = 32 * (NCW + NPROD);
  static constexpr int BAR_BYTES = 1024;   // full/empty of <= 56 ring slots, E full/empty
  static constexpr int FIXED_BYTES = BAR_BYTES + (TMAE ? DE * E_BYTES
                                                       : WAVE ? Geom1<R, NDIM, NCW, VY>::STAGE_BYTES : 0);
};

// Is any table entry (sorted by plane) on planes [z0, z1) in row y, columns [x0, x1)?
__device__ __forceinline__ bool row_has_entry(const int* begin, const int4* ent, int z0, int z1,
                                              int y, int x0, int x1) {
  const int b = __ldg(begin + z0), e = __ldg(begin + z1);
  for (int i = b; i < e; ++i) {
    const int4 t = __ldg(ent + i);
    if (t.y == y && t.x >= x0 && t.x < x1) return true;
  }
  return false;
}

// MODE 0: plain sweep.  MODE 1 (SAVE): this pass also stores u^{n+1} into the snapshot field
// p.outS (stencil_run_save).  MODE 2 (PUSH): fused halo push (band planes into the neighbours'
// ghost zones, producer waits for theirs).  Separate instances, so the plain sweep carries no
// snapshot or push logic in its step body (measured: the push checks cost C4 11 %).
// ISO: isotropic-weight instance (see accumulate), launched when p.iso (3-D, r >= 7, MODE 0).
template <int R, bool WAVE, int NDIM, int NCW, int VY, int MODE, bool ISO = false>
__global__ void __launch_bounds__(Geom1E<R, NDIM, NCW, VY, WAVE>::NTHREADS, 1)
sweep1_kernel(const __grid_constant__ KernelMaps maps, const __grid_constant__ SweepParams p,
              const int nslot) {
  const CUtensorMap& tmapC = maps.u;
  using GE = Geom1E<R, NDIM, NCW, VY, WAVE>;
  constexpr bool TMAE = GE::TMAE;
  constexpr int DE = GE::DE, EB = GE::E_BYTES;
  constexpr bool SAVE = MODE == 1, PUSH = MODE == 2;
  using G = Geom1<R, NDIM, NCW, VY>;
  constexpr int RZ = G::RZ, QN = G::QN, RX2 = G::RX2, RXB = G::RXB, BW = G::BW;
  constexpr int SLOT_F = G::SLOT_BYTES / 4;
  constexpr int PD = G::PD, STAGE_F = G::STAGE_F;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nslot;
  uint64_t* efull = full + 112;                  // E ring barriers (TMAE), bytes 896..1023
  uint64_t* eempty = efull + 8;
  volatile uint32_t* eflag = reinterpret_cast<volatile uint32_t*>(efull + 4);   // per E entry: a == -1 (DE = 4)
  float* ring = reinterpret_cast<float*>(smem + GE::FIXED_BYTES);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * G::OX, ty0 = blockIdx.y * G::OY;
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;
  const int p_first = zb - RZ;
  const int n_arr = (ze - 1 + RZ) - p_first + 1;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 32 * NCW);   // every consumer lane arrives
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
      const uint32_t ebase = static_cast<uint32_t>(__cvta_generic_to_shared(smem + GE::BAR_BYTES));
      const long long fl_stride = (long long)p.fl_nty * p.fl_ntx;
      const unsigned char* fl = p.aflag + zb * fl_stride + (long long)blockIdx.y * p.fl_ntx + blockIdx.x;
      uint32_t f_next = ld_flag(fl);
      for (int s = zb; s < ze; ++s) {
        const uint32_t f = f_next;                       // 1: a == -1 on this tile's plane s
        fl += fl_stride;
        if (s + 1 < ze) f_next = ld_flag(fl);            // in flight across the wait below
        if (s - zb >= DE) mbar_wait(&eempty[es], eph ^ 1u);
        eflag[es] = f;                                   // released to the consumers by the arrive
        mbar_expect_tx(&efull[es], (uint32_t)((f ? 2 : 3) * 64 * GE::OY * 4));   // OOB zero-filled
        const uint32_t fb = static_cast<uint32_t>(__cvta_generic_to_shared(&efull[es]));
        tma_load_3d_e(ebase + es * EB, &maps.p0, fb, tx0, ty0, s - p.zv_lo);
        tma_load_3d_e(ebase + es * EB + GE::E_FIELD, &maps.a0, fb, tx0, ty0, s - p.zv_lo);
        if (!f) tma_load_3d_e(ebase + es * EB + 2 * GE::E_FIELD, &maps.a1, fb, tx0, ty0, s - p.zv_lo);
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
        if (a >= nslot) mbar_wait(&empty[slot], ph ^ 1u);
        if (PUSH) wait_ghost(p, p_first + a, lo_done, hi_done);   // neighbour's push landed
        mbar_expect_tx(&full[slot], (uint32_t)(BW * G::BH * 4));
        tma_load_3d(ring + (size_t)slot * SLOT_F, &tmapC, &full[slot], tx0 - RXB, ty0 - R,
                    p_first + a - p.zv_lo);
        if (++slot == nslot) { slot = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  // warp w owns rows ty0 + w*VY + j (j < VY), a column pair per lane
  const int x0 = tx0 + 2 * lane;
  const int y0 = ty0 + warp * VY;
  const bool xin0 = x0 < p.nx, xin1 = x0 + 1 < p.nx;
  const uint64_t xmask = (xin0 ? 0xffffffffull : 0ull) | (xin1 ? 0xffffffff00000000ull : 0ull);
  bool yin[VY];
  uint64_t mask[VY];
  bool any_row = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    yin[j] = y0 + j < p.ny;                       // warp-uniform
    mask[j] = yin[j] ? xmask : 0ull;
    any_row |= yin[j];
  }
  const bool act = any_row && xin0;               // this lane owns >= 1 interior point
  // warp-uniform: every row and column of this warp is interior (the common case) -> plain stores
  const bool whole = (tx0 + 64 <= p.nx) && (y0 + VY <= p.ny);
  // fused halo push (CTA-uniform): this chunk produces planes of the lo / hi band
  const bool push_lo = PUSH && p.push_lo != nullptr && zb < p.band_lo;
  const bool push_hi = PUSH && p.push_hi != nullptr && ze > p.band_hi;
  const bool push_any = push_lo || push_hi;
  const int col = (warp * VY + R) * BW + 2 * lane + RXB;   // my first row's pair in a ring slot
  const uint64_t DT = splat(p.dt);
  // rare events of this warp's rows (sources / receivers), decided once per CTA chunk
  bool wsrc = false, wrec = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    if (yin[j]) {
      wsrc |= row_has_entry(p.src_begin, p.src, zb, ze, y0 + j, tx0, tx0 + 64);
      wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + j, tx0, tx0 + 64);
    }
  }

  // u^{n-1} and the medium {a,a,c,c} of plane s are staged into per-warp shared memory with
  // cp.async PD planes ahead (no registers held across steps, no wait on fresh loads).
  // Every plane of [zb, ze) lies inside the global domain (host invariant), so each step computes.
  const long long plane = p.plane;
  const int X = p.X, X2 = p.X >> 1;
  float* stage = reinterpret_cast<float*>(smem + GE::BAR_BYTES) + (size_t)warp * (PD + 1) * STAGE_F;
  const int s0 = zb - 2 * RZ;                       // level-0 plane of arrival 0
  const float* gP = p.P + (long long)zb * plane + (long long)y0 * X + x0;   // plane zb
  const float4* gA = p.ac + (long long)zb * (plane >> 1) + (long long)y0 * X2 + (x0 >> 1);
  float* out = p.outP + (long long)zb * plane + (long long)y0 * X + x0;
  float* outs = SAVE ? p.outS + (long long)zb * plane + (long long)y0 * X + x0 : nullptr;   // snapshot
  int q_iss = zb;                                   // next plane to stage
  int e_use = 0, e_iss = 0;                         // staging entries of plane s and of q_iss
  auto stage_next = [&]() {                         // stage plane q_iss (if in the chunk)
    if (q_iss < ze && act) {
      float* e = stage + e_iss * STAGE_F;
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (yin[j]) {
          cp_async8(e + j * 64 + 2 * lane, gP + j * X);
          cp_async16(e + VY * 64 + j * 128 + 4 * lane, gA + j * X2);
        }
      }
    }
    cp_async_commit();
    gP += plane; gA += plane >> 1; ++q_iss;
    if (++e_iss == PD + 1) e_iss = 0;
  };
  if (WAVE && !TMAE) {
#pragma unroll 1
    for (int i = 0; i < PD; ++i) stage_next();
  }
  const float* e_slot = reinterpret_cast<const float*>(smem + GE::BAR_BYTES);
  const int e_pv = (warp * VY) * 64 + 2 * lane;
  const int e_c = GE::E_FIELD / 4 + e_pv, e_a = 2 * (GE::E_FIELD / 4) + e_pv;
  const uint64_t NEG1 = splat(-1.0f);
  int es = 0;
  uint32_t eph = 0;

  uint64_t qn[QN][VY];
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) qn[i][j] = 0ull;
  int slot_a = 0, slot_s = RZ % nslot; // ring slots of the arriving plane and of the centre plane
                                       // (the first centre, plane zb, is arrival RZ)
  uint32_t ph_a = 0;

  // ST_ROT1: the z-queue is rotated by register moves after every step (code = one step body)
  // instead of unrolling the loop by the queue length (code = QN step bodies).
  constexpr int UNR = ST_ROT1 ? 1 : QN;
  for (int base = 0; base < n_arr; base += UNR) {
#pragma unroll
    for (int uu = 0; uu < UNR; ++uu) {
      const int u = ST_ROT1 ? QN - 1 : uu;
      const int idx = base + uu;
      if (idx < n_arr) {
        mbar_wait(&full[slot_a], ph_a);
#pragma unroll
        for (int j = 0; j < VY; ++j) qn[u][j] = lds64(ring + slot_a * SLOT_F + col + j * BW);
        if (idx < RZ) {
          // planes below zb are never a centre: release the slot at once, but only after this
          // lane's loads from it have returned (an LDS can sit behind the cp.async burst in the
          // MIO queue long enough for the producer's next TMA into the slot to land first)
          uint32_t z = 0;
#pragma unroll
          for (int j = 0; j < VY; ++j) z |= zero_after(qn[u][j], p.zero);
          mbar_arrive(&empty[slot_a] + z);
        }
        if (idx >= 2 * RZ) {                          // step s = s0 + idx in [zb, ze)
          if (WAVE && !TMAE) stage_next();            // plane s + PD
          const int s = s0 + idx;
          const float* rp = ring + slot_s * SLOT_F + col;
          uint64_t acc[VY];
          accumulate<R, RZ, QN, VY, NDIM, BW, ISO>(acc, qn, rp, p, md<QN>(u - RZ));
          if (wsrc) {
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yin[j]) acc[j] = add_sources_row(acc[j], p, s, y0 + j, x0, p.wl_step);
          }
          uint64_t o[VY];
          if (TMAE) {
            mbar_wait(&efull[es], eph);
            const float* e = e_slot + es * (EB / 4);
            const uint32_t aneg = eflag[es];        // a == -1 on this plane of the tile: no a box
            uint32_t z = aneg & p.zero;
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c = qn[md<QN>(u - RZ)][j];
              const uint64_t pv = lds64(e + e_pv + j * 64);
              const uint64_t cv = lds64(e + e_c + j * 64);
              uint64_t av = NEG1;
              if (!aneg) av = lds64(e + e_a + j * 64);
              z |= zero_after(pv | cv | av, p.zero);
              o[j] = f2fma(cv, acc[j], f2fma(av, f2sub(pv, c), c)) & mask[j];
            }
            mbar_arrive(&eempty[es] + z);    // release the entry once my loads from it have returned
            if (++es == DE) { es = 0; eph ^= 1u; }
          } else if (WAVE) {
            cp_async_wait<PD>();                      // the group of plane s has landed
            const float* st_e = stage + e_use * STAGE_F;
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c = qn[md<QN>(u - RZ)][j];
              const uint64_t pv = lds64(st_e + j * 64 + 2 * lane);
              const float4 m4 = *reinterpret_cast<const float4*>(st_e + VY * 64 + j * 128 + 4 * lane);
              o[j] = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c)) & mask[j];
            }
            if (++e_use == PD + 1) e_use = 0;
          } else {
#pragma unroll
            for (int j = 0; j < VY; ++j) o[j] = f2fma(DT, acc[j], qn[md<QN>(u - RZ)][j]) & mask[j];
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
          mbar_arrive(&empty[slot_s]);
          if (++slot_s == nslot) slot_s = 0;
          out += plane;
          if (SAVE) outs += plane;
        }
        if (++slot_a == nslot) { slot_a = 0; ph_a ^= 1u; }
        if (ST_ROT1) {
#pragma unroll
          for (int i = 0; i + 1 < QN; ++i)
#pragma unroll
            for (int j = 0; j < VY; ++j) qn[i][j] = qn[i + 1][j];
        }
      }
    }
  }
  if (WAVE && !TMAE) cp_async_wait<0>();
  if (PUSH) signal_peers(p, push_lo, push_hi, 32 * NCW);
}

}  // namespace st
