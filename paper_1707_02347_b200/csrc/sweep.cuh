// sweep.cuh -- temporally blocked 2.5-D star-stencil sweep for sm_100a.
//
// One CTA owns an x-y output tile (OX x OY) and streams the z axis.  Per z step it
//   * receives the next u^n plane (box = tile + level halos + radius) by TMA into a ring of
//     shared-memory slots (mbarrier-tracked, OOB boxes zero-filled = Dirichlet boundary),
//   * keeps every thread's own column of each time level in a register queue of 2r+1 planes
//     (z neighbours never touch shared memory),
//   * evaluates TK time levels: level l computes plane s - l*r (the paper's skew of the
//     time-tiled band by the stencil radius, P:1196-1202 / P:1445 "skew = 4*time", applied
//     here to the streamed axis as a wavefront lag) over an x-y region that shrinks by r per
//     level (overlapped tiles: the redundant halo work replaces the paper's sequential
//     skewed tile order, which would serialise the 148 SMs),
//   * writes only the last two levels (u^{n+TK-1}, u^{n+TK}) to HBM.
// With TK = 1 this is the untiled sweep (Devito's space-only blocking).
//
// Thread mapping: lane -> a PAIR of adjacent x columns (packed fp32x2: FFMA2/FADD2, one
// instruction updates both points bit-identically to two scalar ops); warp -> VY rows.
// Arithmetic follows the canonical per-point order of include/stencil.h exactly, so every
// value is bit-identical to the CPU oracle (oracle/, never included here).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace st {

constexpr int kMaxR = 8;

struct SweepParams {
  int nx, ny;                 // interior extents (x, y)
  int X;                      // row pitch in floats (multiple of 32)
  long long plane;            // X * Y floats per plane
  int gz_lo, gz_hi;           // array planes inside the GLOBAL interior [gz_lo, gz_hi)
  int zv_lo, zv_hi;           // array planes covered by the tensor maps [zv_lo, zv_hi)
  int out_lo, out_hi;         // planes this pass must produce (last level)
  int zchunk;                 // output planes per CTA (gridDim.z chunks)
  const float* P;             // u^{n-1}
  const float* C;             // u^n (also read through the tensor map)
  float* outP;                // TK==1: u^{n+1} (may alias P); TK>1: u^{n+TK-1}
  float* outC;                // TK>1: u^{n+TK}
  float* outS;                // snapshot of this pass's last level (same layout), or nullptr
  const float4* ac;           // medium {a(x),a(x+1),c(x),c(x+1)} per column pair; row = X/2 float4
  // planar-medium kernels (KernelEntry::askip): one byte per (array plane, tile row, tile column),
  // 1 where a == -1 at every interior point of the tile's plane (no damping there: the a box is
  // not loaded), index (z * fl_nty + tile_y) * fl_ntx + tile_x
  const unsigned char* aflag;
  int fl_ntx, fl_nty;
  int write_prev;             // TK>1 heat: also write u^{n+TK-1}
  unsigned zero;              // always 0 (see zero_after)
  float K0, dt;
  float W[3][kMaxR + 1];      // W[axis][k]
  // sources (array-plane sorted): entries (x, y, plane, original index)
  const int* src_begin;       // [Z+1]
  const int4* src;
  const float* wavelet;       // [step][nsrc_total]
  int wl_stride;
  long long wl_step;          // global step index of level 0 of this pass
  // receivers (owned, array-plane sorted)
  const int* rec_begin;       // [Z+1]
  const int4* rec;
  float* trace;               // [run step][nrec_total]
  int tr_stride;
  int tr_step;                // run-relative step index of level 0 of this pass
  // fused halo push (z-slabs, T_c = T_k = 1).  Output planes
  // s < band_lo are also stored at push_lo + (same offset) -- the lo neighbour's output field,
  // pre-shifted by +nzl planes so the store lands in its upper ghost zone; s >= band_hi at
  // push_hi (pre-shifted by -nzl planes, the hi neighbour's lower ghost zone).  A CTA that pushed
  // adds 1 to sig_lo / sig_hi (the neighbour's inbound counter) after its stores, release at
  // system scope.  Before the TMA load of a ghost plane below out_lo (above out_hi) the producer
  // waits until *wait_lo >= wait_lo_target (*wait_hi >= wait_hi_target), acquire at system scope.
  // All pointers nullptr (band_lo = INT_MIN, band_hi = INT_MAX) when not fused.
  float* push_lo;
  float* push_hi;
  int band_lo, band_hi;
  unsigned long long* sig_lo;
  unsigned long long* sig_hi;
  const unsigned long long* wait_lo;
  const unsigned long long* wait_hi;
  unsigned long long wait_lo_target, wait_hi_target;
  int iso;                    // W[0][k] == W[1][k] == W[2][k] bitwise for every k (isotropic dx)
  // two-role exchange pass (sweepx.cuh): tile table (XTile[]), ticket counter, per-tile
  // progress (base + stored-up-to plane, compared modulo 2^32), fault word of timed-out waits
  const void* x_tiles;
  int x_ntiles;
  unsigned* x_ticket;
  unsigned x_ticket_base;
  unsigned* x_prog;
  unsigned x_prog_base;
  unsigned* x_fault;
  unsigned long long* x_trace;   // ST_XTRACE builds only: per (tile, plane) event timestamps
};

// Tensor maps of one launch: u = u^n box with halo (every kernel); the time-tiled kernel's
// producer also streams p0 = u^{n-1} and a0 = medium for level 0, u1 = u^n and a1 = medium for
// level 1 (boxes without halo).
struct KernelMaps {
  CUtensorMap u, p0, a0, u1, a1;
};

// ------------------------------------------------------------------ packed fp32x2 (FTZ) ops
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t r; asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
  uint64_t r; asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b) {
  uint64_t r; asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r; asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ float fadd_ftz(float a, float b) {
  float r; asm("add.rn.ftz.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ float lo_of(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi_of(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t splat(float w) { return pack2(w, w); }

// 0, computed from v and the runtime zero p.zero (so neither nvcc nor ptxas can fold it): adding
// it to an address makes the consumer of that address wait for v (e.g. an LDS result).
__device__ __forceinline__ uint32_t zero_after(uint64_t v, uint32_t zero) {
  uint32_t z;
  asm volatile("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tand.b32 %0, lo, %2;\n\t}"
               : "=r"(z) : "l"(v), "r"(zero));
  return z;
}

__device__ __forceinline__ uint64_t lds64(const float* p) {
  return *reinterpret_cast<const uint64_t*>(p);
}
__device__ __forceinline__ void sts64(float* p, uint64_t v) {
  *reinterpret_cast<uint64_t*>(p) = v;
}

// ------------------------------------------------------------------ mbarrier / TMA
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    // suspend-time hint: the warp sleeps in hardware until the phase completes (no spin issue)
    asm volatile("{\n\t.reg .pred q;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, 0x989680;\n\t"
                 "selp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  } while (!ok);
}
// ---- programmatic dependent launch (PDL): a sweep launched with programmatic stream
// serialisation may start while the previous kernel of the stream drains.  Every CTA lets the
// next launch begin once it is running (launch_dependents) and, before touching any global data,
// waits until the previous grid has completed and its memory is visible (wait).  Only the
// prologue (barrier init, tensor-map prefetch) and the launch latency overlap the predecessor.
__device__ __forceinline__ void pdl_prologue_done() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---- fused halo push: cross-GPU signalling (system scope)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* a, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" :: "l"(a), "l"(v) : "memory");
}
// Wait until a neighbour's pushes of the previous step have landed, then order the later TMA
// (async-proxy) reads of the ghost planes after that acquire.
// A neighbour that never signals (a mismatched run sequence) must not hang the GPU: after ~20 s
// the kernel traps, the run fails with ST_ECUDA and the plan enters ST_ESTATE.
__device__ __forceinline__ void wait_peer(const unsigned long long* ctr, unsigned long long target) {
  if (ld_acquire_sys(ctr) < target) {
    const long long t0 = clock64();
    while (ld_acquire_sys(ctr) < target) {
      __nanosleep(256);
      if (clock64() - t0 > 40000000000ll) __trap();
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Producer side of every untiled kernel: before the TMA load of array plane z.
__device__ __forceinline__ void wait_ghost(const SweepParams& p, int z, bool& lo_done, bool& hi_done) {
  if (!lo_done && z < p.out_lo) {
    if (p.wait_lo) wait_peer(p.wait_lo, p.wait_lo_target);
    lo_done = true;
  }
  if (!hi_done && z >= p.out_hi) {
    if (p.wait_hi) wait_peer(p.wait_hi, p.wait_hi_target);
    hi_done = true;
  }
}
// Consumer side, after the CTA's last step: every pushing thread fences its peer stores, the
// consumer warps meet at named barrier 1, one thread bumps the neighbours' counters.
__device__ __forceinline__ void signal_peers(const SweepParams& p, bool pushed_lo, bool pushed_hi,
                                             int nconsumer_threads) {
  if (!(pushed_lo || pushed_hi)) return;   // CTA-uniform
  __threadfence_system();
  asm volatile("bar.sync 1, %0;" :: "r"(nconsumer_threads) : "memory");
  if (threadIdx.x == 0) {
    if (pushed_lo) red_release_sys_add(p.sig_lo, 1ull);
    if (pushed_hi) red_release_sys_add(p.sig_hi, 1ull);
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
         "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------ compile-time geometry
template <int R, int TK>
struct Halo {
  // x half-width of level l's region beyond the output tile, kept even so column pairs never
  // straddle a region edge: hx(TK-1) = 0, hx(l) = round_up(hx(l+1) + R, 2).
  static constexpr int hx(int l) { return l >= TK - 1 ? 0 : ((hx(l + 1) + R + 1) & ~1); }
  static constexpr int hy(int l) { return R * (TK - 1 - l); }
};

template <int R, int TK, int NDIM, int VY, int NWY>
struct Geom {
  static constexpr int RZ = (NDIM == 3) ? R : 0;   // z radius (2-D: none)
  static constexpr int QN = 2 * RZ + 1;            // register queue length
  static constexpr int RX2 = (R + 1) & ~1;         // x reach of the pair loads, even
  static constexpr int RXB = (R + 3) & ~3;         // x halo of the TMA box, multiple of 4 floats
  static constexpr int GW = 64;                    // grid width (32 lanes x 2 columns)
  static constexpr int GH = NWY * VY;              // grid height
  static constexpr int HX0 = Halo<R, TK>::hx(0);
  static constexpr int HY0 = Halo<R, TK>::hy(0);
  // The TMA box must start on a 16-byte boundary (cuda-gdb: a box starting at x = -6 floats
  // raised "Warp Illegal Instruction" at UTMALDG).  Grid origins are = -HX0 (mod 4), so the box
  // starts XS = HX0 % 4 columns further left and is widened to keep rows a multiple of 32 B.
  static constexpr int XS = HX0 % 4;
  static constexpr int BW = GW + 2 * RXB + (XS ? 8 : 0);   // TMA box width (multiple of 8 floats)
  static constexpr int BH = GH + 2 * R;            // TMA box height
  static constexpr int BCOL = RXB + XS;            // column of grid x = 0 inside the box
  static constexpr int OX = GW - 2 * HX0;          // output tile
  static constexpr int OY = GH - 2 * HY0;
  static constexpr int SLOT_BYTES = ((BW * BH * 4) + 127) / 128 * 128;
  static constexpr int LVL_FLOATS = GW * (GH + 2 * R);   // one level plane buffer, R pad rows
                                                         // above/below (rows of a warp outside a
                                                         // level's region read them, results masked)
  static constexpr int NTHREADS = 32 * NWY;
  static_assert(OX > 0 && OY > 0, "tile too small for this radius / depth");
  static_assert(BW <= 256 && BH <= 256, "TMA box limit");
};

template <int QN>
__device__ __forceinline__ constexpr int md(int a) { return ((a % QN) + QN) % QN; }

// shared-memory bytes for nslot ring slots
template <int R, int TK, int NDIM, int VY, int NWY>
__host__ __device__ constexpr size_t sweep_smem_bytes(int nslot) {
  using G = Geom<R, TK, NDIM, VY, NWY>;
  return 128 /* barriers */ + (size_t)nslot * G::SLOT_BYTES +
         (TK > 1 ? (size_t)2 * (TK - 1) * G::LVL_FLOATS * 4 : 0);
}

// Canonical accumulation for the VY rows of one thread at one level (see stencil.h):
//   acc = K0*c; for k: acc = fma(Wx_k, left+right, acc); fma(Wy_k, ...); fma(Wz_k, ...)
// rowp  : smem pointer of (my first row, my column pair) in the in-plane buffer of this level
// PITCH : floats per smem row;  q : the z-queue of this level's INPUT, center at index CI.
template <int R, int RZ, int QN, int VY, int NDIM, int PITCH, bool ISO = false>
__device__ __forceinline__ void accumulate(uint64_t (&acc)[VY], const uint64_t (&q)[QN][VY],
                                           const float* rowp, const SweepParams& p, const int CI) {
  constexpr int RX2 = (R + 1) & ~1;
  const uint64_t K0 = splat(p.K0);
#pragma unroll
  for (int j = 0; j < VY; ++j) {
    const float* rp = rowp + j * PITCH;
    const uint64_t c = q[CI][j];
    uint64_t A[RX2 + 1];   // aligned pairs (2m, 2m+1) relative to my pair, m = -RX2/2..RX2/2
#pragma unroll
    for (int m = -RX2 / 2; m <= RX2 / 2; ++m) A[m + RX2 / 2] = (m == 0) ? c : lds64(rp + 2 * m);
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
      const uint64_t yl = (j - k >= 0) ? q[CI][(j - k) >= 0 ? (j - k) : 0] : lds64(rp - k * PITCH);
      const uint64_t yr = (j + k < VY) ? q[CI][(j + k) < VY ? (j + k) : 0] : lds64(rp + k * PITCH);
      // ISO (launched only when W[0][k] == W[1][k] == W[2][k] bitwise, p.iso): one weight per k,
      // so the r weights stay in uniform registers instead of being re-loaded every step
      a = f2fma(splat(p.W[ISO ? 0 : 1][k]), f2add(yl, yr), a);
      if (NDIM == 3)
        a = f2fma(splat(p.W[ISO ? 0 : 2][k]), f2add(q[md<QN>(CI - k)][j], q[md<QN>(CI + k)][j]), a);
    }
    acc[j] = a;
  }
}

// Sources located on plane q (rare): acc += w, in source index order, on the matching element.
template <int VY>
__device__ __forceinline__ void add_sources(uint64_t (&acc)[VY], const SweepParams& p, int q,
                                            int y0, int x0, long long wl_row) {
  const int sb = __ldg(p.src_begin + q), se = __ldg(p.src_begin + q + 1);
  if (sb >= se) return;
  for (int i = sb; i < se; ++i) {
    const int4 e = __ldg(p.src + i);
    const int j = e.y - y0;
    if (j < 0 || j >= VY || (e.x != x0 && e.x != x0 + 1)) continue;
    const float w = __ldg(p.wavelet + wl_row * p.wl_stride + e.w);
#pragma unroll
    for (int jj = 0; jj < VY; ++jj)
      if (jj == j)
        acc[jj] = (e.x == x0) ? pack2(fadd_ftz(lo_of(acc[jj]), w), hi_of(acc[jj]))
                              : pack2(lo_of(acc[jj]), fadd_ftz(hi_of(acc[jj]), w));
  }
}

// Receivers on plane q inside the output tile: trace[row][orig] = value (unique writer).
template <int VY>
__device__ __forceinline__ void sample_receivers(const uint64_t (&val)[VY], const SweepParams& p,
                                                 int q, int y0, int x0, int tx0, int ty0, int ox,
                                                 int oy, int trow) {
  const int rb = __ldg(p.rec_begin + q), re = __ldg(p.rec_begin + q + 1);
  if (rb >= re) return;
  for (int i = rb; i < re; ++i) {
    const int4 e = __ldg(p.rec + i);
    if (e.x < tx0 || e.x >= tx0 + ox || e.y < ty0 || e.y >= ty0 + oy) continue;
    const int j = e.y - y0;
    if (j < 0 || j >= VY || (e.x != x0 && e.x != x0 + 1)) continue;
#pragma unroll
    for (int jj = 0; jj < VY; ++jj)
      if (jj == j)
        p.trace[(long long)trow * p.tr_stride + e.w] = (e.x == x0) ? lo_of(val[jj]) : hi_of(val[jj]);
  }
}

// =========================================================================================
template <int R, int TK, bool WAVE, int NDIM, int VY, int NWY>
__global__ void __launch_bounds__(32 * NWY, 1)
sweep_kernel(const __grid_constant__ CUtensorMap tmapC, const __grid_constant__ SweepParams p,
             const int nslot) {
  using G = Geom<R, TK, NDIM, VY, NWY>;
  constexpr int RZ = G::RZ, QN = G::QN, BCOL = G::BCOL, GW = G::GW, GH = G::GH, BW = G::BW;
  constexpr int HX0 = G::HX0, HY0 = G::HY0, OX = G::OX, OY = G::OY;
  constexpr int NL = (TK > 1) ? TK - 1 : 1;
  constexpr int SLOT_F = G::SLOT_BYTES / 4;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  float* ring = reinterpret_cast<float*>(smem + 128);
  float* lvl = reinterpret_cast<float*>(smem + 128 + (size_t)nslot * G::SLOT_BYTES);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tx0 = blockIdx.x * OX, ty0 = blockIdx.y * OY;   // output tile origin (interior)
  const int gx = tx0 - HX0, gy = ty0 - HY0;                 // thread-grid origin
  const int x0 = gx + 2 * lane;                             // my column pair (x0, x0+1)
  const int ry = warp * VY;                                 // my first row in the grid
  const int y0 = gy + ry;                                   // my first interior row
  const int zb = p.out_lo + blockIdx.z * p.zchunk;
  const int ze = min(p.out_hi, zb + p.zchunk);
  if (zb >= ze) return;

  // interior masks
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
  const int rowoff = y0 * p.X + x0;        // element offset of (my first row, my pair) in a plane
  const int X2 = p.X >> 1;
  const int acoff = y0 * X2 + (x0 >> 1);   // float4 offset of the same in an ac plane
  const long long acplane = p.plane >> 1;  // float4 per ac plane

  // stream bounds: level l computes plane s - l*RZ
  const int s_first = zb - (TK - 1) * RZ;
  const int s_last = ze - 1 + (TK - 1) * RZ;
  const int p_first = s_first - RZ;
  const int n_arr = (s_last + RZ) - p_first + 1;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int next_issue = 0;   // arrival index of the next TMA to issue (thread 0 only)
  auto issue = [&](int a) {
    const int slot = a % nslot;
    mbar_expect_tx(&bars[slot], (uint32_t)(G::BW * G::BH * 4));
    tma_load_3d(ring + (size_t)slot * SLOT_F, &tmapC, &bars[slot], gx - BCOL, gy - R,
                p_first + a - p.zv_lo);
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmapC)) : "memory");
    for (; next_issue < n_arr && next_issue < nslot; ++next_issue) issue(next_issue);
  }

  uint64_t qn[QN][VY];
  uint64_t ql[NL][QN][VY];
#pragma unroll
  for (int i = 0; i < QN; ++i)
#pragma unroll
    for (int j = 0; j < VY; ++j) {
      qn[i][j] = 0ull;
#pragma unroll
      for (int l = 0; l < NL; ++l) ql[l][i][j] = 0ull;
    }
  const uint64_t DT = splat(p.dt);
  int lbuf = 0;

  for (int base = 0; base < n_arr; base += QN) {
#pragma unroll
    for (int u = 0; u < QN; ++u) {
      const int idx = base + u;
      if (idx < n_arr) {
        const int s = p_first + idx - RZ;             // level-0 plane of this step
        const int slot_a = idx % nslot;
        const uint32_t par_a = (uint32_t)((idx / nslot) & 1);
        bool lv_on[TK];
#pragma unroll
        for (int l = 0; l < TK; ++l) {
          const int q = s - l * RZ;
          lv_on[l] = (idx >= 2 * RZ) && (q >= zb - (TK - 1 - l) * RZ) &&
                     (q < ze + (TK - 1 - l) * RZ) && (q >= p.gz_lo) && (q < p.gz_hi);
        }

        // ---- this step's global loads, issued before the barrier wait -------------------
        uint64_t prev0[VY];
        float4 acv[TK][VY];
        if (WAVE) {
#pragma unroll
          for (int j = 0; j < VY; ++j) prev0[j] = 0ull;
          if (lv_on[0] && xin0) {
            const float* Pq = p.P + (long long)s * p.plane + rowoff;
#pragma unroll
            for (int j = 0; j < VY; ++j)
              if (yin[j]) prev0[j] = __ldg(reinterpret_cast<const unsigned long long*>(Pq + j * p.X));
          }
#pragma unroll
          for (int l = 0; l < TK; ++l) {
#pragma unroll
            for (int j = 0; j < VY; ++j) acv[l][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (lv_on[l] && xin0) {
              const float4* Aq = p.ac + (long long)(s - l * RZ) * acplane + acoff;
#pragma unroll
              for (int j = 0; j < VY; ++j)
                if (yin[j]) acv[l][j] = __ldg(Aq + j * X2);
            }
          }
        }

        // ---- arrival of u^n plane p_first+idx: wait, feed the queue --------------------------
        const float* sa = ring + (size_t)slot_a * SLOT_F + (ry + R) * BW + 2 * lane + BCOL;
        mbar_wait(&bars[slot_a], par_a);
#pragma unroll
        for (int j = 0; j < VY; ++j) qn[u][j] = lds64(sa + j * BW);

        // ---- level 0 at plane s ---------------------------------------------------------
        uint64_t out0[VY];
#pragma unroll
        for (int j = 0; j < VY; ++j) out0[j] = 0ull;
        if (lv_on[0]) {
          const int slot_s = (idx - RZ) % nslot;
          const float* cs = ring + (size_t)slot_s * SLOT_F + (ry + R) * BW + 2 * lane + BCOL;
          uint64_t acc[VY];
          accumulate<R, RZ, QN, VY, NDIM, BW>(acc, qn, cs, p, md<QN>(u - RZ));
          add_sources<VY>(acc, p, s, y0, x0, p.wl_step);
#pragma unroll
          for (int j = 0; j < VY; ++j) {
            const uint64_t c = qn[md<QN>(u - RZ)][j];
            uint64_t o;
            if (WAVE) {
              const float4 m4 = acv[0][j];
              o = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(prev0[j], c), c));
            } else {
              o = f2fma(DT, acc[j], c);
            }
            out0[j] = o & rmask[j];
          }
        }

        if (TK == 1) {
          // ---- write u^{n+1} (in place over u^{n-1}), sample receivers --------------------
          if (lv_on[0] && s >= zb && s < ze) {
            if (xin0) {
              float* dst = p.outP + (long long)s * p.plane + rowoff;
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                if (yin[j]) {
                  if (xin1) sts64(dst + j * p.X, out0[j]);
                  else dst[j * p.X] = lo_of(out0[j]);
                  if (p.outS) {
                    float* sn = p.outS + (long long)s * p.plane + rowoff + j * p.X;
                    if (xin1) sts64(sn, out0[j]); else sn[0] = lo_of(out0[j]);
                  }
                }
              }
            }
            sample_receivers<VY>(out0, p, s, y0, x0, tx0, ty0, OX, OY, p.tr_step);
          }
          __syncthreads();   // the ring slot of plane s may now be recycled
          if (tid == 0 && next_issue < n_arr && next_issue <= idx - RZ + nslot) {
            issue(next_issue);
            ++next_issue;
          }
        } else {
          // ---- time-tiled levels 1..TK-1 ------------------------------------------------
#pragma unroll
          for (int j = 0; j < VY; ++j) ql[0][u][j] = out0[j];
          if (lv_on[0] && s >= zb && s < ze)
            sample_receivers<VY>(out0, p, s, y0, x0, tx0, ty0, OX, OY, p.tr_step);
          float* lb = lvl + (size_t)lbuf * (TK - 1) * G::LVL_FLOATS;
#pragma unroll
          for (int l = 1; l < TK; ++l) {
            // publish level l-1 at plane s - l*RZ (this level's centre plane)
            float* lp = lb + (size_t)(l - 1) * G::LVL_FLOATS + (ry + R) * GW + 2 * lane;
#pragma unroll
            for (int j = 0; j < VY; ++j) sts64(lp + j * GW, ql[l - 1][md<QN>(u - RZ)][j]);
            __syncthreads();
            if (l == 1 && tid == 0 && next_issue < n_arr && next_issue <= idx - RZ + nslot) {
              issue(next_issue);
              ++next_issue;
            }
            const int q = s - l * RZ;
            constexpr int dummy = 0; (void)dummy;
            const int ex = (HX0 - Halo<R, TK>::hx(l)) / 2;      // lanes outside region l
            const int eyl = HY0 - Halo<R, TK>::hy(l);            // grid rows outside region l
            const bool lane_in = (lane >= ex) && (lane < 32 - ex);
            const bool rows_in = (ry + VY > eyl) && (ry < GH - eyl);   // warp-uniform
            uint64_t ol[VY];
#pragma unroll
            for (int j = 0; j < VY; ++j) ol[j] = 0ull;
            if (lv_on[l] && lane_in && rows_in) {
              uint64_t acc[VY];
              accumulate<R, RZ, QN, VY, NDIM, GW>(acc, ql[l - 1], lp, p, md<QN>(u - RZ));
              add_sources<VY>(acc, p, q, y0, x0, p.wl_step + l);
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                const int rr = ry + j;
                const uint64_t c = ql[l - 1][md<QN>(u - RZ)][j];
                uint64_t o;
                if (WAVE) {
                  const uint64_t pv = (l == 1) ? qn[md<QN>(u - 2 * RZ)][j]
                                               : ql[l >= 2 ? l - 2 : 0][md<QN>(u - 2 * RZ)][j];
                  const float4 m4 = acv[l][j];
                  o = f2fma(pack2(m4.z, m4.w), acc[j], f2fma(pack2(m4.x, m4.y), f2sub(pv, c), c));
                } else {
                  o = f2fma(DT, acc[j], c);
                }
                ol[j] = (rr >= eyl && rr < GH - eyl) ? (o & rmask[j]) : 0ull;
              }
            }
            if (l < TK - 1) {
#pragma unroll
              for (int j = 0; j < VY; ++j) ql[l < NL ? l : 0][u][j] = ol[j];
            } else if (lv_on[l] && q >= zb && q < ze && lane_in && rows_in && xin0) {
              // ---- last level: u^{n+TK} and u^{n+TK-1} on the output tile ------------------
              const long long off = (long long)q * p.plane + rowoff;
#pragma unroll
              for (int j = 0; j < VY; ++j) {
                const int rr = ry + j;
                if (rr >= eyl && rr < GH - eyl && yin[j]) {
                  const uint64_t pv = ql[TK - 2][md<QN>(u - RZ)][j];
                  if (xin1) {
                    sts64(p.outC + off + j * p.X, ol[j]);
                    if (WAVE || p.write_prev) sts64(p.outP + off + j * p.X, pv);
                    if (p.outS) sts64(p.outS + off + j * p.X, ol[j]);
                  } else {
                    p.outC[off + j * p.X] = lo_of(ol[j]);
                    if (WAVE || p.write_prev) p.outP[off + j * p.X] = lo_of(pv);
                    if (p.outS) p.outS[off + j * p.X] = lo_of(ol[j]);
                  }
                }
              }
            }
            if (lv_on[l] && q >= zb && q < ze)
              sample_receivers<VY>(ol, p, q, y0, x0, tx0, ty0, OX, OY, p.tr_step + l);
          }
          lbuf ^= 1;
        }
      }
    }
  }
}

}  // namespace st
