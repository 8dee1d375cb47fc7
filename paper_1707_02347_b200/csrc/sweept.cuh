// sweept.cuh -- time-tiled (T_k = 2) 3-D sweep whose tiles exchange their first time level
// through L2 instead of recomputing it (G3).
//
// The paper's time tile computes several time levels of a block of
// points before moving on, skewing the block by the stencil radius per level so that every level
// only needs values the block itself (or an EARLIER block) produced.  On a GPU all
// x-y tiles run at once, so the earlier design (sweep2.cuh) made every tile self-contained by
// recomputing an r-wide halo of level 1 (overlapped tiles, x1.40 work at SO8).  This kernel keeps
// the paper's dependence structure instead: a tile computes level 1 only over its own points,
// stores it (level 1 is an output of the pass anyway: u^{n+1}), publishes per-plane progress, and
// reads the r-wide level-1 halo it needs for level 2 back from its neighbours' stores, which are
// still in L2 because all tiles stream z in step.  HBM traffic is that of the two-level pass
// (read u^{n-1}, u^n, a, c; write u^{n+1}, u^{n+2}: 12 B per update) with no redundant arithmetic
// except at band cuts (below).
//
// CTA = one 64 x H tile (H = NCW*VY rows), all z planes of one chunk:
//   * warp NCW   (producer U): TMA boxes of u^n planes (tile + r halo; OOB zero = Dirichlet) into
//                 a ring of NU slots;
//   * warp NCW+1 (producer X): for every level-1 plane p of the chunk, waits until this CTA's
//                 consumer warps stored it (l1done mbarrier) and the neighbour tiles whose
//                 level-1 values the level-2 halo needs published p (relaxed polls, acquire once
//                 satisfied), then TMA-loads the level-1 box of plane p (tile + r halo) from the
//                 output field into a ring of NB slots;
//   * warp NCW+2 (publisher P): publishes the CTA's level-1 progress (st.release.gpu, whose
//                 MEMBAR.GPU would otherwise stall the box issue);
//   * warps 0..NCW-1 (consumers): warp w owns rows y0 + w*VY + j, a column pair per lane (packed
//                 fp32x2), with TWO register z-queues of 2r+1 planes: u^n (level-1 input) and
//                 the lane's own level-1 results (level-2 input), both 2r+1+D planes long.
//                 Arrival a of plane pa:
//                   level 1 at plane s = pa - r (x/y from the u^n slot, z from the u^n queue),
//                   level 2 at plane q = s - r - D (x/y from the level-1 box, z from the level-1
//                   queue; u^n(q) is the oldest u^n queue entry; a, c(q) kept in the staging
//                   ring).  The lag D beyond the r the stencil needs is slack for the exchange.
//   Both levels follow the canonical per-point order of include/stencil.h, so every stored value
//   is bit-identical to the untiled oracle (oracle/, never included here).
//
// Scheduling and deadlock freedom (host side: abi.cu plan_tiles):
//   * tiles are numbered chunk-major, then band, then row-major; a CTA takes the next tile from a
//     global ticket counter after griddepcontrol.wait, so tiles START in ticket order;
//   * a tile depends on its left/right/below neighbours (same band: later tickets) and on the
//     tile above (same band, or the band above: earlier tickets); a band holds at most as many
//     tiles as can be resident at once, so the earliest unfinished band is always fully resident
//     and finishes (induction), whatever the number of waves;
//   * band cuts: the first tile row of a band starts r rows above the previous band's last level-1
//     row (its top r level-1 rows repeat the previous band's: computed again and stored again with
//     identical bits, so the x-neighbours of those rows come from the same tile row), and the last
//     tile row of a band produces level 2 for H - r rows only -- so a band never waits on a later
//     band (the paper's skew, applied between bands).
//   * every flag wait is bounded (~4 s): on timeout the CTA records a fault (stencil_sync reports
//     it) and continues, so a broken invariant cannot hang the GPU.
#pragma once
#include "sweep1.cuh"

namespace st {

template <int R, int NCW, int VY, bool WAVE, int D>
struct GeomT {
  static constexpr int H = NCW * VY;               // tile rows
  static constexpr int QN = 2 * R + 1 + D;         // z-queue length (2r+1 + level-2 lag D)
  static constexpr int RXB = (R + 3) & ~3;         // box x halo, multiple of 4 floats (16 B)
  static constexpr int BW = 64 + 2 * RXB;
  static constexpr int BH = H + 2 * R;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
  static constexpr int KD = 32;                    // l1done ring (planes)
  static constexpr int BAR_BYTES = 1024;
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int NB = (R + D + 1) < 6 ? (R + D + 1) : 6;   // level-1 box ring (lookahead <= r+D)
  static constexpr int PD = 3;                     // cp.async staging distance (planes)
  static constexpr int NPE = PD + 1;               // u^{n-1} staging entries
  static constexpr int NAE = PD + 1 + R + D;       // a/c staging entries (kept r+D planes for level 2)
  static constexpr int STP_F = VY * 64;            // floats per u^{n-1} entry (per warp)
  static constexpr int STA_F = VY * 128;           // floats per a/c entry (per warp)
  static constexpr int STAGE_BYTES = WAVE ? NCW * (NPE * STP_F + NAE * STA_F) * 4 : 0;
  static constexpr int fixed() { return BAR_BYTES + STAGE_BYTES + NB * SLOT_BYTES; }
  // u^n ring: r+1 planes in use + prefetch, as deep as shared memory allows (<= r+1+4)
  static constexpr int NU_MAX = (SMEM_MAX - fixed()) / SLOT_BYTES;
  static constexpr int NU = NU_MAX < R + 5 ? NU_MAX : R + 5;
  static constexpr bool OK = NU >= R + 2;
  static constexpr int SMEM = fixed() + NU * SLOT_BYTES;
  static constexpr int NTHREADS = 32 * (NCW + 3);
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
  static_assert(H >= 2 * R, "band cuts need tile rows >= 2r");
};

// ---- inter-CTA progress (generic proxy, gpu scope)
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cta_shared(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(a)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_shared(unsigned* a, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" :: "r"(smem_u32(a)), "r"(v) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred q;\n\t"
               "mbarrier.test_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, q;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

#ifdef ST_XTRACE
// diagnostic builds: globaltimer stamps per (tile, plane, event), ST_XTRACE_K planes per tile
#define ST_XTRACE_K 1024
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define XT(ev, k)                                                                              \
  do {                                                                                         \
    if (p.x_trace && (k) >= 0 && (k) < ST_XTRACE_K)                                            \
      p.x_trace[((size_t)me * ST_XTRACE_K + (k)) * 12 + (ev)] = gtimer();                       \
  } while (0)
#else
#define XT(ev, k) do {} while (0)
#endif

template <int R, bool WAVE, int NCW, int VY, int D>
__global__ void __launch_bounds__(32 * (NCW + 3), 1)
sweept_kernel(const __grid_constant__ CUtensorMap tmapU, const __grid_constant__ CUtensorMap tmapL,
              const __grid_constant__ SweepParams p) {
  using G = GeomT<R, NCW, VY, WAVE, D>;
  static_assert(G::OK, "exchange kernel does not fit in shared memory");
  constexpr int QN = G::QN, BW = G::BW, BH = G::BH, RXB = G::RXB, H = G::H;
  constexpr int NU = G::NU, NB = G::NB, KD = G::KD, PD = G::PD, NPE = G::NPE, NAE = G::NAE;
  constexpr int STP_F = G::STP_F, STA_F = G::STA_F;
  constexpr int SLOT_F = G::SLOT_BYTES / 4;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* ufull = reinterpret_cast<uint64_t*>(smem);
  uint64_t* uempty = ufull + NU;
  uint64_t* bfull = uempty + NU;
  uint64_t* bempty = bfull + NB;
  uint64_t* l1done = bempty + NB;
  int* tile_sh = reinterpret_cast<int*>(l1done + KD);
  unsigned* kown_sh = reinterpret_cast<unsigned*>(tile_sh + 1);   // level-1 planes stored (X -> P)
  float* stage0 = reinterpret_cast<float*>(smem + G::BAR_BYTES);
  float* bring = reinterpret_cast<float*>(smem + G::BAR_BYTES + G::STAGE_BYTES);
  float* uring = bring + NB * SLOT_F;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int i = 0; i < NU; ++i) { mbar_init(&ufull[i], 1); mbar_init(&uempty[i], 32 * NCW); }
    for (int i = 0; i < NB; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 32 * NCW); }
    for (int i = 0; i < KD; ++i) mbar_init(&l1done[i], NCW);
    fence_mbar_init();
  }
  pdl_prologue_done();
  if (tid == 0) {
    *tile_sh = (int)(atomicAdd(p.x_ticket, 1u) - p.x_ticket_base);
    *kown_sh = 0u;
  }
  __syncthreads();
  const int me = *tile_sh;
  if (me >= p.x_ntiles) return;
  const TileDesc td = p.x_tiles[me];
  const int tx0 = td.x0, ty0 = td.y0;
  const int zb = td.zb, ze = td.ze;
  const int n_load = (ze - zb) + 4 * R;     // u^n planes zb-2r .. ze+2r-1
  const int n_arr = n_load + D;             // + D steps that only finish level 2
  const int pa0 = zb - 2 * R;

  if (warp == NCW) {
    // ---------------------------------------------------------------- producer U: u^n planes
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapU)) : "memory");
      int slot = 0;
      uint32_t ph = 0;
      for (int a = 0; a < n_load; ++a) {
        if (a >= NU) mbar_wait(&uempty[slot], ph ^ 1u);
        mbar_expect_tx(&ufull[slot], (uint32_t)(BW * BH * 4));
        tma_load_3d(uring + (size_t)slot * SLOT_F, &tmapU, &ufull[slot], tx0 - RXB, ty0 - R,
                    pa0 + a - p.zv_lo);
        if (++slot == NU) { slot = 0; ph ^= 1u; }
      }
    }
    return;
  }
  if (warp == NCW + 2) {
    // ---------------------------------------------------------------- publisher P
    // Publishes how many level-1 planes this CTA has stored.  The release store (MEMBAR.GPU:
    // the consumers' stores, observed through l1done, become visible first) stalls only this warp.
    if (lane == 0) {
      // progress source: producer X's count of observed l1done phases (shared word, release/
      // acquire at CTA scope), so this warp never waits on an mbarrier phase it could alias
      const unsigned base = p.x_prog_base;
      const int n = ze - zb;
      int k = 0;
      while (k < n) {
        const int c = (int)ld_acquire_cta_shared(kown_sh);
        if (c > k) {
          k = c;
          st_release_gpu_u32(p.x_prog + me, base + (unsigned)k);
#ifdef ST_XTRACE
          for (int kk = 0; kk < k; ++kk) if (p.x_trace[((size_t)me * ST_XTRACE_K + kk) * 12 + 8] == 0) XT(8, kk);
#endif
        } else {
          __nanosleep(32);
        }
      }
    }
    return;
  }
  if (warp == NCW + 1) {
    // ---------------------------------------------------------------- producer X: level-1 boxes
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapL)) : "memory");
      // Box(k) = the level-1 plane zb+k of this tile plus its r halo, read back from the output
      // field once (a) this CTA's consumers stored plane k (l1done) and (b) every neighbour tile
      // published >= k+1 planes.  Polls are relaxed (one L2 round trip for all pending
      // neighbours); a satisfied neighbour is re-read with ld.acquire (synchronises with its
      // release), then fence.proxy.async orders the generic-proxy view before the TMA read.
      // Boxes run up to NB planes ahead of the consumers, who need box(q) r+D planes after
      // level 1 of q was stored, so the exchange latency hides behind r+D planes of compute.
      const unsigned base = p.x_prog_base;
      const int n = ze - zb;
      int slot = 0;
      uint32_t ph = 0;
      int kown = 0, kbox = 0;
      int seen[4];
      bool need[4];
#pragma unroll
      for (int d = 0; d < 4; ++d) { seen[d] = 0; need[d] = td.dep[d] >= 0; }
      bool ok = true;
      long long t_idle = clock64();
      XT(6, 0);
      while (kbox < n) {
        bool moved = false;
        const int kown0 = kown;
        if (kbox == kown) {                         // nothing to do until level 1 of kbox is stored
          mbar_wait(&l1done[kown % KD], (uint32_t)((kown / KD) & 1));
          XT(0, kown);
          ++kown;
        }
        while (kown < n && mbar_test(&l1done[kown % KD], (uint32_t)((kown / KD) & 1))) {
          XT(0, kown);
          ++kown;
        }
        if (kown > kown0) st_release_cta_shared(kown_sh, (unsigned)kown);
        bool ready = true;
#ifdef ST_XNODEP
        ok = false;   // diagnostic: ignore the neighbours (wrong results, pipeline speed only)
#endif
        if (ok) {
          unsigned v[4];
#pragma unroll
          for (int d = 0; d < 4; ++d)
            if (need[d] && seen[d] <= kbox) v[d] = ld_relaxed_gpu_u32(p.x_prog + td.dep[d]);
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            if (need[d] && seen[d] <= kbox) {
              int rel = (int)(v[d] - base);
              if (rel > kbox) rel = (int)(ld_acquire_gpu_u32(p.x_prog + td.dep[d]) - base);
              if (rel > seen[d]) seen[d] = rel;
              if (seen[d] <= kbox) ready = false;
            }
          }
        }
        if (ready) {
          XT(1, kbox);
          if (kbox < NB || mbar_test(&bempty[slot], ph ^ 1u)) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            mbar_expect_tx(&bfull[slot], (uint32_t)(BW * BH * 4));
            tma_load_3d(bring + (size_t)slot * SLOT_F, &tmapL, &bfull[slot], tx0 - RXB, ty0 - R,
                        zb + kbox - p.zv_lo);
            XT(2, kbox);
            if (++slot == NB) { slot = 0; ph ^= 1u; }
            ++kbox;
            moved = true;
          }
        }
        if (moved) {
          t_idle = clock64();
        } else {
          __nanosleep(32);
          if (clock64() - t_idle > 8000000000ll) {   // a neighbour never progressed: give up
            atomicExch(p.x_fault, 1u);                 // waiting (results invalid, no hang)
            ok = false;
            t_idle = clock64();
          }
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
  bool yin[VY], yst[VY], yl2[VY];
  uint64_t mask[VY];
  bool any_row = false;
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    const int y = y0 + j;
    yin[j] = y >= 0 && y < p.ny;                        // warp-uniform
    yst[j] = yin[j] && y >= td.st_lo && y < td.st_hi;   // level-1 stored by this tile
    yl2[j] = yin[j] && y >= td.l2_lo && y < td.l2_hi;   // level 2 produced by this tile
    mask[j] = yin[j] ? xmask : 0ull;
    any_row |= yin[j];
  }
  const bool act = any_row && xin0;
  const bool xwhole = tx0 + 64 <= p.nx;
  const int col = (warp * VY + R) * BW + 2 * lane + RXB;   // my first row's pair in a box slot
  const uint64_t DT = splat(p.dt);
  bool wsrc = false, wrec = false;
  const int zs0 = max(0, zb - R), zs1 = min(p.gz_hi, ze + R);   // level-1 planes (array, clamped)
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    if (yin[j]) {
      if (zs0 < zs1) wsrc |= row_has_entry(p.src_begin, p.src, zs0, zs1, y0 + j, tx0, tx0 + 64);
      if (yl2[j]) wrec |= row_has_entry(p.rec_begin, p.rec, zb, ze, y0 + j, tx0, tx0 + 64);
    }
  }

  const long long plane = p.plane;
  const int X = p.X, X2 = p.X >> 1;
  // staging: u^{n-1} (NPE entries) and a/c (NAE entries) of level-1 plane s, PD planes ahead
  float* stP = stage0 + (size_t)warp * (NPE * STP_F + NAE * STA_F);
  float* stA = stP + NPE * STP_F;
  const int s_first = zb - R;                             // first level-1 plane
  const float* gP = p.P + (long long)s_first * plane + (long long)y0 * X + x0;
  const float4* gA = p.ac + (long long)s_first * (plane >> 1) + (long long)y0 * X2 + (x0 >> 1);
  int q_iss = s_first;
  int eP_iss = 0, eA_iss = 0, eP_use = 0, eA_use = 0;
  auto stage_next = [&]() {
    if (q_iss >= p.zv_lo && q_iss < p.zv_hi && q_iss < ze + R && act) {
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (yin[j]) {
          cp_async8(stP + eP_iss * STP_F + j * 64 + 2 * lane, gP + j * X);
          cp_async16(stA + eA_iss * STA_F + j * 128 + 4 * lane, gA + j * X2);
        }
      }
    }
    cp_async_commit();
    gP += plane; gA += plane >> 1; ++q_iss;
    if (++eP_iss == NPE) eP_iss = 0;
    if (++eA_iss == NAE) eA_iss = 0;
  };
  if (WAVE) {
#pragma unroll 1
    for (int i = 0; i < PD; ++i) stage_next();
  }

  float* out1 = p.outP + (long long)zb * plane + (long long)y0 * X + x0;   // level 1, plane zb
  float* out2 = p.outC + (long long)zb * plane + (long long)y0 * X + x0;   // level 2, plane zb

  uint64_t qn[QN][VY], q1[QN][VY];
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) { qn[i][j] = 0ull; q1[i][j] = 0ull; }

  int slot_a = 0, slot_c = 0;          // u^n ring: arriving plane, level-1 centre plane
  uint32_t ph_a = 0;
  int slot_b = 0;                      // level-1 box ring
  uint32_t ph_b = 0;

  auto store_rows = [&](float* d, const uint64_t (&o)[VY], const bool (&rows)[VY]) {
    if (xwhole) {
#pragma unroll
      for (int j = 0; j < VY; ++j)
        if (rows[j]) sts64(d + j * X, o[j]);
    } else if (xin0) {
#pragma unroll
      for (int j = 0; j < VY; ++j) {
        if (rows[j]) {
          if (xin1) sts64(d + j * X, o[j]);
          else d[j * X] = lo_of(o[j]);
        }
      }
    }
  };

  int eA2 = R % NAE;                   // a/c staging entry of level-2 plane q (first: zb)
#pragma unroll 1
  for (int base = 0; base < n_arr; base += QN) {
#pragma unroll
    for (int uu = 0; uu < QN; ++uu) {
      const int a = base + uu;
      if (a < n_arr) {
        if (a < n_load) {
          mbar_wait(&ufull[slot_a], ph_a);
#pragma unroll
          for (int j = 0; j < VY; ++j) qn[uu][j] = lds64(uring + slot_a * SLOT_F + col + j * BW);
          if (a < R) {
            // planes below the first level-1 centre: never a centre, release once the loads returned
            uint32_t z = 0;
#pragma unroll
            for (int j = 0; j < VY; ++j) z |= zero_after(qn[uu][j], p.zero);
            mbar_arrive(&uempty[slot_a] + z);
            if (++slot_c == NU) slot_c = 0;
          }
        }
        if (a >= 2 * R && a < n_load) {
          // ---------------- level 1 at plane s (queue entry of s: (uu - 2r) mod QN)
          const int s = pa0 + a - R;
          if (WAVE) stage_next();                       // plane s + PD
          const bool sin = s >= p.gz_lo && s < p.gz_hi;   // inside the global interior
          uint64_t acc[VY];
          accumulate<R, R, QN, VY, 3, BW>(acc, qn, uring + slot_c * SLOT_F + col, p, md<QN>(uu - R));
          if (wsrc && sin) {
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yin[j]) acc[j] = add_sources_row(acc[j], p, s, y0 + j, x0, p.wl_step);
          }
          uint64_t o[VY];
          if (WAVE) {
            cp_async_wait<PD>();
            const float* eP = stP + eP_use * STP_F;
            const float* eA = stA + eA_use * STA_F;
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c = qn[md<QN>(uu - R)][j];
              const uint64_t pv = lds64(eP + j * 64 + 2 * lane);
              const float4 m4 = *reinterpret_cast<const float4*>(eA + j * 128 + 4 * lane);
              o[j] = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c)) & mask[j];
            }
            if (++eP_use == NPE) eP_use = 0;
            if (++eA_use == NAE) eA_use = 0;
          } else {
#pragma unroll
            for (int j = 0; j < VY; ++j) o[j] = f2fma(DT, acc[j], qn[md<QN>(uu - R)][j]) & mask[j];
          }
#pragma unroll
          for (int j = 0; j < VY; ++j) {
            if (!sin) o[j] = 0ull;
            q1[md<QN>(uu - 2 * R)][j] = o[j];
          }
          const bool own = s >= zb && s < ze;
          if (own) {
            store_rows(out1, o, yst);
            if (wrec) {
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yl2[j]) sample_receivers_row(o[j], p, s, y0 + j, x0, p.tr_step);
            }
            out1 += plane;
            __syncwarp();
            if (lane == 0) mbar_arrive(&l1done[(s - zb) % KD]);
            if (warp == 0 && lane == 0) XT(5, s - zb);
          }
          mbar_arrive(&uempty[slot_c]);
          if (++slot_c == NU) slot_c = 0;
        }
        if (a >= 4 * R + D) {
          // -------------- level 2 at plane q = s - r - D (its level-1 queue entry: (uu - 3r - D))
          const int q = pa0 + a - 2 * R - D;
          if (warp == 0 && lane == 0) XT(7, q - zb);
          mbar_wait(&bfull[slot_b], ph_b);
          if (warp == 0 && lane == 0) XT(3, q - zb);
          uint64_t acc2[VY];
          accumulate<R, R, QN, VY, 3, BW>(acc2, q1, bring + slot_b * SLOT_F + col, p, md<QN>(uu - 3 * R - D));
          if (wsrc) {
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yin[j]) acc2[j] = add_sources_row(acc2[j], p, q, y0 + j, x0, p.wl_step + 1);
          }
          uint64_t o2[VY];
          if (WAVE) {
            const float* eA = stA + eA2 * STA_F;
            if (++eA2 == NAE) eA2 = 0;
#pragma unroll
            for (int j = 0; j < VY; ++j) {
              const uint64_t c1 = q1[md<QN>(uu - 3 * R - D)][j];
              const uint64_t un = qn[md<QN>(uu - 2 * R - D)][j];   // u^n(q): the oldest u^n entry
              const float4 m4 = *reinterpret_cast<const float4*>(eA + j * 128 + 4 * lane);
              o2[j] = f2fma(pack2(m4.z, m4.w), acc2[j], f2fma(pack2(m4.x, m4.y), f2sub(un, c1), c1)) & mask[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < VY; ++j) o2[j] = f2fma(DT, acc2[j], q1[md<QN>(uu - 3 * R - D)][j]) & mask[j];
          }
          store_rows(out2, o2, yl2);
          if (p.outS) store_rows(p.outS + (out2 - p.outC), o2, yl2);   // stencil_run_save
          if (wrec) {
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yl2[j]) sample_receivers_row(o2[j], p, q, y0 + j, x0, p.tr_step + 1);
          }
          out2 += plane;
          if (warp == 0 && lane == 0) XT(4, q - zb);
          mbar_arrive(&bempty[slot_b]);
          if (++slot_b == NB) { slot_b = 0; ph_b ^= 1u; }
        }
        if (a < n_load && ++slot_a == NU) { slot_a = 0; ph_a ^= 1u; }
      }
    }
  }
  if (WAVE) cp_async_wait<0>();
}

}  // namespace st
