// sweepx.cuh -- time-tiled (T_k = 2) pass as TWO untiled sweeps in one launch, level 1 feeding
// level 2 through L2 (G3).
//
// The paper's time tile computes two (or more) time levels of a block before moving on, so the
// second level reads the first from fast memory instead of DRAM, and
// skews the block by the stencil radius per level so every level only needs values produced
// EARLIER.  Here the "block" is a z-streamed x-y tile and the fast memory is the
// 126 MB L2: a launch holds two kinds of tiles,
//   * L1 tiles: an untiled sweep u^n -> u^{n+1} (reads u^{n-1}, u^n, a, c from HBM, writes u^{n+1}),
//     publishing after every plane how many planes they have stored (never waiting on anyone);
//   * L2 tiles: an untiled sweep u^{n+1} -> u^{n+2} over the same grid, skewed r rows up, whose
//     TMA producer waits before each u^{n+1} plane until the L1 tiles covering that plane's box
//     published it; its u^{n+1}, u^n (as "u_prev") and a, c reads hit L2 because it trails the L1
//     tiles by a few planes.
// HBM traffic per update: (16 + 4 + 4) B / 2 = 12 B (vs 20 B untiled).  Both roles are the
// warp-specialised untiled sweep of sweep1.cuh (TMA ring of u boxes, register z-queue, packed
// fp32x2, canonical per-point order of include/stencil.h -> bit-identical to the oracle).
//
// Scheduling (host: abi.cu plan_xtiles): tiles are numbered L1 row 0, L2 row 0, L1 row 1, L2
// row 1, ... (chunk-major); a CTA takes the next number from a ticket counter after
// griddepcontrol.wait, so tiles START in ticket order.  An L2 tile of row j needs the L1 tiles of
// rows j-1, j (and their x-neighbours) -- all earlier tickets -- and L1 tiles wait on nothing, so
// no tile ever waits on one that has not started: deadlock-free for any grid size or wave count.
// z-chunks: the L1 tiles of a chunk also compute the r planes on each side (redundantly, same
// bits), so a chunk's L2 tiles only depend on their own chunk.
// Every wait is bounded (~4 s): on timeout the tile records a fault (stencil_sync reports it) and
// continues, so a broken invariant cannot hang the GPU.
#pragma once
#include "sweep1.cuh"

namespace st {

struct XTile {                // one tile of an L1/L2 exchange pass (built by abi.cu plan_xtiles)
  int x0, y0;                 // tile origin (interior coords), 64 x (NCW*VY) points
  int role;                   // 0: level 1 (publishes), 1: level 2 (waits)
  int zb, ze;                 // planes this tile computes and stores, array coords
  int oz0, oz1;               // planes whose receiver samples this tile owns
  int nd;                     // L2: number of L1 tiles it waits on
  int dep[9];                 // L2: L1 tiles whose boxes cover this tile's u^{n+1} box
  int partner;                // L1: the L2 tile of the same column and row index (throttle), or -1
};

// Optional throttle (off by default, ST_XLAG = 0): an L1 tile waits before loading plane p until
// its partner L2 tile (if started) stored p - XLAG, bounding the L2 re-read window.  Measured
// slower at every window tried (C3 T_k=2: 250 GPts/s without, 176 at 48, 117 at 32, 63 at 16)
// because it couples every L1 tile to the publication latency of the L2 tiles.
// A window must exceed the L2 tile's own lag, ~2r + its ring prefetch, or the pass stalls.
#ifndef ST_XLAG
#define ST_XLAG 0
#endif

__device__ __forceinline__ unsigned ldx_relaxed_gpu(const unsigned* a) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ldx_acquire_gpu(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stx_release_gpu(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ldx_acquire_cta_shared(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(a)) : "memory");
  return v;
}
__device__ __forceinline__ void stx_release_cta_shared(unsigned* a, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" :: "r"(smem_u32(a)), "r"(v) : "memory");
}

#ifdef ST_XTRACE
#define ST_XTRACE_K 1024
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// diagnostic builds: per (tile, plane-index k = plane - zb) stamps of %globaltimer:
//   0 publisher saw all warps stored k, 1 release store of k+1 returned (L1 and L2 tiles),
//   2 L2 producer starts waiting for plane zb+k-r... (its arrival k), 3 condition satisfied,
//   4 L1 producer throttle wait start, 5 throttle satisfied, 6 tile start (k = 0)
#define XS(ev, k)                                                                              \
  do {                                                                                         \
    if (p.x_trace && (k) >= 0 && (k) < ST_XTRACE_K)                                            \
      p.x_trace[((size_t)me * ST_XTRACE_K + (k)) * 12 + (ev)] = gtimer();                      \
  } while (0)
#else
#define XS(ev, k) do {} while (0)
#endif

// ---- L2 eviction hints: data the L2 tiles re-read stays (evict_last), data nobody re-reads in
// this pass leaves first (evict_first), so the re-read window fits the 126 MB L2
#ifndef ST_XHINT
#define ST_XHINT 1
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int c0, int c1, int c2, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
         "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void cp_async8_hint(float* dst, const float* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;"
               :: "r"(smem_u32(dst)), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(float* dst, const float4* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
               :: "r"(smem_u32(dst)), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void st64_hint(float* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" :: "l"(p), "l"(v), "l"(pol) : "memory");
}

template <int R, bool WAVE, int NCW, int VY>
__global__ void __launch_bounds__(32 * (NCW + 2), 1)
sweepx_kernel(const __grid_constant__ CUtensorMap tmapU, const __grid_constant__ CUtensorMap tmapL,
              const __grid_constant__ SweepParams p, const int nslot) {
  using G = Geom1<R, 3, NCW, VY>;
  constexpr int QN = G::QN, RXB = G::RXB, BW = G::BW;
  constexpr int SLOT_F = G::SLOT_BYTES / 4;
  constexpr int PD = G::PD, STAGE_F = G::STAGE_F;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + nslot;
  unsigned* wprog = reinterpret_cast<unsigned*>(empty + nslot);   // per consumer warp: planes stored
  int* tile_sh = reinterpret_cast<int*>(wprog + NCW);
  float* ring = reinterpret_cast<float*>(smem + ((16 * nslot + 4 * NCW + 4 + 127) / 128) * 128);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 32 * NCW);
    }
    for (int i = 0; i < NCW; ++i) wprog[i] = 0u;
    fence_mbar_init();
  }
  pdl_prologue_done();
  if (tid == 0) *tile_sh = (int)(atomicAdd(p.x_ticket, 1u) - p.x_ticket_base);
  __syncthreads();
  const int me = *tile_sh;
  if (me >= p.x_ntiles) return;
  const XTile td = static_cast<const XTile*>(p.x_tiles)[me];
  const bool L2 = td.role == 1;
  const CUtensorMap* tmap = L2 ? &tmapL : &tmapU;
  const int tx0 = td.x0, ty0 = td.y0;
  const int zb = td.zb, ze = td.ze;
  const int p_first = zb - R;
  const int n_arr = (ze - zb) + 2 * R;
  const unsigned base = p.x_prog_base;
  const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();

  if (warp == NCW) {
    // ------------------------------------------------------------------ producer warp
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
      int slot = 0;
      uint32_t ph = 0;
      // L2: the smallest "stored up to plane" the L1 deps published so far (absolute planes)
      int seen_min = 0;
      int thr_seen = -(1 << 30);                     // L1: partner progress seen (absolute)
      bool ok = true;
      for (int a = 0; a < n_arr; ++a) {
        if (a >= nslot) mbar_wait(&empty[slot], ph ^ 1u);
        const int pl = p_first + a;                  // array plane of this box
        if (ST_XLAG > 0 && !L2 && ok && td.partner >= 0 && pl - ST_XLAG >= thr_seen) {
          // throttle: wait until the partner L2 tile stored plane pl - XLAG, if it has started
          // (a partner that has not published in this launch reads below base: no wait)
          const long long t0 = clock64();
          XS(4, a);
          while (true) {
            const int v = (int)(ldx_relaxed_gpu(p.x_prog + td.partner) - base);
            if (v < 0 || v > pl - ST_XLAG) { thr_seen = v < 0 ? thr_seen : v; XS(5, a); break; }
            __nanosleep(128);
            if (clock64() - t0 > 8000000000ll) { atomicExch(p.x_fault, 1u); ok = false; break; }
          }
        }
#ifdef ST_XNODEP
        ok = false;   // diagnostic: no waits at all (wrong results, pipeline/L2 bound only)
#endif
        if (L2 && ok && pl >= p.gz_lo && pl < p.gz_hi) {
          // every dep must have stored planes up to pl: published (absolute) >= pl + 1
          const int need = pl + 1;
          if (seen_min < need) {
            const long long t0 = clock64();
            XS(2, a);
            while (true) {
              unsigned v[9];
#pragma unroll
              for (int d = 0; d < 9; ++d)
                if (d < td.nd) v[d] = ldx_relaxed_gpu(p.x_prog + td.dep[d]);
              int mn = 1 << 30;
#pragma unroll
              for (int d = 0; d < 9; ++d)
                if (d < td.nd) mn = min(mn, (int)(v[d] - base));
              if (mn >= need) {
#pragma unroll
                for (int d = 0; d < 9; ++d)        // synchronise with each dep's release
                  if (d < td.nd) (void)ldx_acquire_gpu(p.x_prog + td.dep[d]);
                seen_min = mn;
                XS(3, a);
                break;
              }
              __nanosleep(64);
              if (clock64() - t0 > 8000000000ll) {   // an L1 tile never progressed: give up
                atomicExch(p.x_fault, 1u);           // waiting (results invalid, no hang)
                ok = false;
                break;
              }
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        mbar_expect_tx(&full[slot], (uint32_t)(BW * G::BH * 4));
        if (ST_XHINT)   // L1: u^n box (re-read by L2 tiles) stays; L2: u^{n+1} box read last
          tma_load_3d_hint(ring + (size_t)slot * SLOT_F, tmap, &full[slot], tx0 - RXB, ty0 - R,
                           pl - p.zv_lo, L2 ? pol_first : pol_last);
        else
          tma_load_3d(ring + (size_t)slot * SLOT_F, tmap, &full[slot], tx0 - RXB, ty0 - R,
                      pl - p.zv_lo);
        if (++slot == nslot) { slot = 0; ph ^= 1u; }
      }
    }
    return;
  }
  if (warp == NCW + 1) {
    // ------------------------------------------------------------------ publisher
    // min over the consumer warps of "planes stored" -> st.release.gpu (its MEMBAR.GPU makes
    // the consumers' stores visible first and stalls only this warp).  Values are absolute:
    // base + (last stored plane + 1); an L2 tile publishes base + zb at once ("started").
    if (lane == 0) {
      const int n = ze - zb;
      int done = 0;
      XS(6, 0);
      if (L2) stx_release_gpu(p.x_prog + me, base + (unsigned)zb);
      while (done < n) {
        int mn = n;
        for (int w = 0; w < NCW; ++w) mn = min(mn, (int)ldx_acquire_cta_shared(wprog + w));
        if (mn > done) {
#ifdef ST_XTRACE
          for (int kk = done; kk < mn; ++kk) XS(0, kk);
#endif
          const int d0 = done;
          done = mn;
          stx_release_gpu(p.x_prog + me, base + (unsigned)(zb + done));   // stored < zb + done
#ifdef ST_XTRACE
          for (int kk = d0; kk < done; ++kk) XS(1, kk);
#else
          (void)d0;
#endif
        } else {
          __nanosleep(64);
        }
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
    yin[j] = y0 + j >= 0 && y0 + j < p.ny;         // warp-uniform
    mask[j] = yin[j] ? xmask : 0ull;
    any_row |= yin[j];
  }
  const bool act = any_row && xin0;
  const bool whole = (tx0 + 64 <= p.nx) && (y0 >= 0) && (y0 + VY <= p.ny);
  const int col = (warp * VY + R) * BW + 2 * lane + RXB;
  const uint64_t DT = splat(p.dt);
  // the level this tile computes: L1 = step wl_step (trace row tr_step), L2 = the next one
  const long long wl_step = p.wl_step + (L2 ? 1 : 0);
  const int tr_step = p.tr_step + (L2 ? 1 : 0);
  // receivers: owned planes only (a chunk's L1 tiles also compute r planes on each side)
  const int rz0 = max(td.oz0, p.out_lo), rz1 = min(td.oz1, p.out_hi);
  bool wsrc = false, wrec = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    if (yin[j]) {
      wsrc |= row_has_entry(p.src_begin, p.src, max(zb, p.gz_lo), min(ze, p.gz_hi), y0 + j, tx0, tx0 + 64);
      if (rz0 < rz1) wrec |= row_has_entry(p.rec_begin, p.rec, rz0, rz1, y0 + j, tx0, tx0 + 64);
    }
  }

  const long long plane = p.plane;
  const int X = p.X, X2 = p.X >> 1;
  float* stage = ring + (size_t)nslot * SLOT_F + (size_t)warp * (PD + 1) * STAGE_F;
  const float* srcP = L2 ? p.C : p.P;              // "u_prev" of this level: u^{n-1} or u^n
  float* dst = L2 ? p.outC : p.outP;               // u^{n+1} or u^{n+2}
  const float* gP = srcP + (long long)zb * plane + (long long)y0 * X + x0;
  const float4* gA = p.ac + (long long)zb * (plane >> 1) + (long long)y0 * X2 + (x0 >> 1);
  float* out = dst + (long long)zb * plane + (long long)y0 * X + x0;
  int q_iss = zb;
  int e_use = 0, e_iss = 0;
  auto stage_next = [&]() {
    if (q_iss < ze && act) {
      float* e = stage + e_iss * STAGE_F;
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (yin[j]) {
          if (ST_XHINT) {   // L1: u^{n-1} dead after this read, a/c re-read by L2 tiles
            cp_async8_hint(e + j * 64 + 2 * lane, gP + j * X, L2 ? pol_first : pol_first);
            cp_async16_hint(e + VY * 64 + j * 128 + 4 * lane, gA + j * X2, L2 ? pol_first : pol_last);
          } else {
            cp_async8(e + j * 64 + 2 * lane, gP + j * X);
            cp_async16(e + VY * 64 + j * 128 + 4 * lane, gA + j * X2);
          }
        }
      }
    }
    cp_async_commit();
    gP += plane; gA += plane >> 1; ++q_iss;
    if (++e_iss == PD + 1) e_iss = 0;
  };
  if (WAVE) {
#pragma unroll 1
    for (int i = 0; i < PD; ++i) stage_next();
  }

  uint64_t qn[QN][VY];
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) qn[i][j] = 0ull;
  int slot_a = 0, slot_s = R % nslot;
  uint32_t ph_a = 0;
  const int s0 = zb - 2 * R;
  int stored = 0;

  for (int base_i = 0; base_i < n_arr; base_i += QN) {
#pragma unroll
    for (int uu = 0; uu < QN; ++uu) {
      const int idx = base_i + uu;
      if (idx < n_arr) {
        mbar_wait(&full[slot_a], ph_a);
#pragma unroll
        for (int j = 0; j < VY; ++j) qn[uu][j] = lds64(ring + slot_a * SLOT_F + col + j * BW);
        if (idx < R) {
          uint32_t z = 0;
#pragma unroll
          for (int j = 0; j < VY; ++j) z |= zero_after(qn[uu][j], p.zero);
          mbar_arrive(&empty[slot_a] + z);
        }
        if (idx >= 2 * R) {
          if (WAVE) stage_next();
          const int s = s0 + idx;
          const float* rp = ring + slot_s * SLOT_F + col;
          uint64_t acc[VY];
          accumulate<R, R, QN, VY, 3, BW>(acc, qn, rp, p, md<QN>(uu - R));
          const bool sin = s >= p.gz_lo && s < p.gz_hi;
          if (wsrc && sin) {
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yin[j]) acc[j] = add_sources_row(acc[j], p, s, y0 + j, x0, wl_step);
          }
          uint64_t o[VY];
          if (WAVE) {
            cp_async_wait<PD>();
            const float* st_e = stage + e_use * STAGE_F;
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c = qn[md<QN>(uu - R)][j];
              const uint64_t pv = lds64(st_e + j * 64 + 2 * lane);
              const float4 m4 = *reinterpret_cast<const float4*>(st_e + VY * 64 + j * 128 + 4 * lane);
              o[j] = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c)) & mask[j];
            }
            if (++e_use == PD + 1) e_use = 0;
          } else {
#pragma unroll
            for (int j = 0; j < VY; ++j) o[j] = f2fma(DT, acc[j], qn[md<QN>(uu - R)][j]) & mask[j];
          }
          if (sin) {
            if (whole) {
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                if (ST_XHINT) st64_hint(out + j * X, o[j], L2 ? pol_first : pol_last);
                else sts64(out + j * X, o[j]);
              }
            } else if (act) {
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                if (yin[j]) {
                  if (xin1) sts64(out + j * X, o[j]);
                  else out[j * X] = lo_of(o[j]);
                }
              }
            }
            if (L2 && p.outS) {                    // stencil_run_save: snapshot of level 2
              float* so = p.outS + (out - p.outC);
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yin[j] && xin0) {
                  if (xin1) sts64(so + j * X, o[j]);
                  else so[j * X] = lo_of(o[j]);
                }
            }
            if (wrec && s >= rz0 && s < rz1) {
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yin[j]) sample_receivers_row(o[j], p, s, y0 + j, x0, tr_step);
            }
          }
          {                                         // publish: this warp stored plane s
            ++stored;
            __syncwarp();
            if (lane == 0) stx_release_cta_shared(wprog + warp, (unsigned)stored);
          }
          mbar_arrive(&empty[slot_s]);
          if (++slot_s == nslot) slot_s = 0;
          out += plane;
        }
        if (++slot_a == nslot) { slot_a = 0; ph_a ^= 1u; }
      }
    }
  }
  if (WAVE) cp_async_wait<0>();
}

}  // namespace st
