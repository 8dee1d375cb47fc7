// registry.h -- compiled kernel instances (one per (ndim, time_order, radius, t_kernel)).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <utility>

#include "sweep.cuh"
#include "sweep1.cuh"
#include "sweep1s.cuh"
#include "sweep2.cuh"
#include "sweepx.cuh"
#include "sweeph.cuh"

#ifndef ST_T1_DEPTH
#define ST_T1_DEPTH 6   // untiled kernel: ring planes of prefetch beyond the radius+1 in use
#endif

namespace st {

typedef cudaError_t (*launch_fn)(const KernelMaps& maps, const SweepParams& p, dim3 grid,
                                 int nslot, size_t smem, cudaStream_t stream);
typedef cudaError_t (*attr_fn)(size_t smem, cudaFuncAttributes* attr, int* blocks_per_sm,
                               int nthreads);

struct KernelEntry {
  int ndim, time_order, radius, tk;
  int vy, nwy, nthreads;
  int ox, oy;          // output tile
  int bw, bh;          // TMA box
  int rz;              // z radius (0 in 2-D)
  size_t slot_bytes;   // one ring slot
  size_t fixed_bytes;  // barriers + level buffers
  launch_fn launch;
  attr_fn query;       // sets max dynamic smem, returns attributes and occupancy
  int extra_depth;     // preferred ring prefetch depth beyond the rz+1 resident planes
  int ebw = 0, eh0 = 0, eh1 = 0;   // time-tiled kernel (wave): field box width, level-0 / level-1
                                   // box rows of the producer-streamed u^{n-1}, u^n, medium
  int fixed_slots = 0;             // > 0: the ring depth is compiled in (sweep1s_kernel)
  int askip = 0;                   // 1: planar medium (maps.a0 = c box, maps.a1 = a box) and
                                   //    SweepParams::aflag (a-box loads skipped where a == -1)
  int exch = 0;                    // 1: two-role exchange pass (sweepx.cuh): host builds a tile
                                   //    table; maps.u1 = u^{n+1} box map over the level-1 output
};

// Defined in the generated instance translation units.
const KernelEntry* registry_begin();
const KernelEntry* registry_end();
const KernelEntry* find_kernel(int ndim, int time_order, int radius, int tk);

template <int R, int TK, bool WAVE, int NDIM, int VY, int NWY>
cudaError_t launch_sweep(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                         size_t smem, cudaStream_t stream) {
  sweep_kernel<R, TK, WAVE, NDIM, VY, NWY><<<grid, 32 * NWY, smem, stream>>>(maps.u, p, nslot);
  return cudaGetLastError();
}

template <int R, int TK, bool WAVE, int NDIM, int VY, int NWY>
cudaError_t query_sweep(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweep_kernel<R, TK, WAVE, NDIM, VY, NWY>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

template <int R, int TK, bool WAVE, int NDIM, int VY, int NWY>
constexpr KernelEntry make_entry() {
  using G = Geom<R, TK, NDIM, VY, NWY>;
  return KernelEntry{NDIM, WAVE ? 2 : 1, R, TK, VY, NWY, G::NTHREADS, G::OX, G::OY, G::BW, G::BH,
                     G::RZ, (size_t)G::SLOT_BYTES,
                     (size_t)128 + (TK > 1 ? (size_t)2 * (TK - 1) * G::LVL_FLOATS * 4 : 0),
                     &launch_sweep<R, TK, WAVE, NDIM, VY, NWY>,
                     &query_sweep<R, TK, WAVE, NDIM, VY, NWY>, 3};
}

#ifndef ST_PDL
#define ST_PDL 1        // untiled sweeps launch with programmatic stream serialisation (sweep.cuh)
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, int block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = ST_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- warp-specialised untiled kernel (sweep1.cuh)
template <int R, bool WAVE, int NDIM, int NCW, int VY>
cudaError_t launch_sweep1(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                          size_t smem, cudaStream_t stream) {
  const int block = Geom1E<R, NDIM, NCW, VY, WAVE>::NTHREADS;
  if (p.outS)
    return launch_pdl(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 1>, grid, block, smem, stream, maps, p, nslot);
  if (p.push_lo || p.push_hi || p.wait_lo || p.wait_hi) {
    if constexpr (NDIM == 3)
      return launch_pdl(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 2>, grid, block, smem, stream, maps, p, nslot);
    else
      return cudaErrorNotSupported;
  }
  if constexpr (NDIM == 3 && R >= 7) {   // measured: C4 SO16 239 -> 245 GPts/s; SO12 unchanged
    if (p.iso)
      return launch_pdl(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 0, true>, grid, block, smem, stream, maps, p, nslot);
  }
  return launch_pdl(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 0>, grid, block, smem, stream, maps, p, nslot);
}

template <int R, bool WAVE, int NDIM, int NCW, int VY>
cudaError_t query_sweep1(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweep1_kernel<R, WAVE, NDIM, NCW, VY, 0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 1>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if constexpr (NDIM == 3) {
    e = cudaFuncSetAttribute(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if constexpr (NDIM == 3 && R >= 7) {
    e = cudaFuncSetAttribute(sweep1_kernel<R, WAVE, NDIM, NCW, VY, 0, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

template <int R, bool WAVE, int NDIM, int NCW, int VY = 1>
constexpr KernelEntry make_entry1() {
  using G = Geom1<R, NDIM, NCW, VY>;
  using GE = Geom1E<R, NDIM, NCW, VY, WAVE>;
  KernelEntry e{NDIM, WAVE ? 2 : 1, R, 1, VY, NCW, GE::NTHREADS, G::OX, G::OY, G::BW, G::BH,
                G::RZ, (size_t)G::SLOT_BYTES, (size_t)GE::FIXED_BYTES,
                &launch_sweep1<R, WAVE, NDIM, NCW, VY>, &query_sweep1<R, WAVE, NDIM, NCW, VY>, ST_T1_DEPTH};
  if (GE::TMAE) { e.ebw = 64; e.eh0 = GE::OY; e.eh1 = GE::OY; e.askip = 1; }   // host encodes the u^{n-1} / medium maps
  return e;
}

// ---- untiled kernel with a compiled-in ring of 2r+1 slots (sweep1s.cuh)
template <int R, bool WAVE, int NCW, int VY>
cudaError_t launch_sweep1s(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                           size_t smem, cudaStream_t stream) {
  const int block = Geom1S<R, NCW, VY, WAVE>::NTHREADS;
  if (p.outS)
    return launch_pdl(sweep1s_kernel<R, WAVE, NCW, VY, 1>, grid, block, smem, stream, maps, p, nslot);
  if (p.push_lo || p.push_hi || p.wait_lo || p.wait_hi)
    return launch_pdl(sweep1s_kernel<R, WAVE, NCW, VY, 2>, grid, block, smem, stream, maps, p, nslot);
  if constexpr (R >= 7) {
    if (p.iso)
      return launch_pdl(sweep1s_kernel<R, WAVE, NCW, VY, 0, true>, grid, block, smem, stream, maps, p, nslot);
  }
  return launch_pdl(sweep1s_kernel<R, WAVE, NCW, VY, 0>, grid, block, smem, stream, maps, p, nslot);
}

template <int R, bool WAVE, int NCW, int VY>
cudaError_t query_sweep1s(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweep1s_kernel<R, WAVE, NCW, VY, 0>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  for (auto kk : {sweep1s_kernel<R, WAVE, NCW, VY, 1>, sweep1s_kernel<R, WAVE, NCW, VY, 2>}) {
    e = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if constexpr (R >= 7) {
    e = cudaFuncSetAttribute(sweep1s_kernel<R, WAVE, NCW, VY, 0, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

template <int R, bool WAVE, int NCW, int VY>
constexpr KernelEntry make_entry1s() {
  using G = Geom1<R, 3, NCW, VY>;
  using S = Geom1S<R, NCW, VY, WAVE>;
  KernelEntry e{3, WAVE ? 2 : 1, R, 1, VY, NCW, S::NTHREADS, G::OX, G::OY, G::BW, G::BH,
                R, (size_t)S::SLOT_BYTES, (size_t)S::FIXED_BYTES,
                &launch_sweep1s<R, WAVE, NCW, VY>, &query_sweep1s<R, WAVE, NCW, VY>, S::NS - R - 1};
  e.fixed_slots = S::NS;
  if (S::TMAE) { e.ebw = 64; e.eh0 = S::OY; e.eh1 = S::OY; e.askip = 1; }   // host encodes the u^{n-1} / medium maps
  return e;
}

// ---- warp-specialised time-tiled kernel (sweep2.cuh): one warp group per level
template <int R, int TK, bool WAVE, int OY>
cudaError_t launch_sweep2(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                          size_t smem, cudaStream_t stream) {
  constexpr int block = Geom2<R, TK, WAVE, OY>::NTHREADS;
  if (p.outS) return launch_pdl(sweep2_kernel<R, TK, WAVE, OY, true>, grid, block, smem, stream, maps, p, nslot);
  return launch_pdl(sweep2_kernel<R, TK, WAVE, OY, false>, grid, block, smem, stream, maps, p, nslot);
}

template <int R, int TK, bool WAVE, int OY>
cudaError_t query_sweep2(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweep2_kernel<R, TK, WAVE, OY, false>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sweep2_kernel<R, TK, WAVE, OY, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

#ifndef ST_T2_DEPTH
#define ST_T2_DEPTH 3   // time-tiled kernel: ring planes of prefetch beyond the radius+1 in use
#endif

template <int R, int TK, bool WAVE, int OY>
constexpr KernelEntry make_entry2() {
  using G = Geom2<R, TK, WAVE, OY>;
  return KernelEntry{3, WAVE ? 2 : 1, R, TK, 2, G::NCW, G::NTHREADS, G::OX, G::OY, G::BW, G::BH,
                     R, (size_t)G::SLOT_BYTES, (size_t)G::FIXED_BYTES,
                     &launch_sweep2<R, TK, WAVE, OY>, &query_sweep2<R, TK, WAVE, OY>, ST_T2_DEPTH,
                     WAVE ? G::EBW : 0, WAVE ? G::GH : 0, WAVE ? G::OY : 0};
}

// ---- two-role exchange pass (sweepx.cuh): T_k = 2 as L1 + L2 untiled sweeps through L2
template <int R, bool WAVE, int NCW, int VY>
cudaError_t launch_sweepx(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                          size_t smem, cudaStream_t stream) {
  return launch_pdl(sweepx_kernel<R, WAVE, NCW, VY>, grid, 32 * (NCW + 2), smem, stream, maps.u, maps.u1, p, nslot);
}

template <int R, bool WAVE, int NCW, int VY>
cudaError_t query_sweepx(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweepx_kernel<R, WAVE, NCW, VY>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

template <int R, bool WAVE, int NCW, int VY>
constexpr KernelEntry make_entryX() {
  using G = Geom1<R, 3, NCW, VY>;
  KernelEntry e{3, WAVE ? 2 : 1, R, 2, VY, NCW, 32 * (NCW + 2), G::OX, G::OY, G::BW, G::BH,
                R, (size_t)G::SLOT_BYTES, (size_t)1024 + (WAVE ? G::STAGE_BYTES : 0),
                &launch_sweepx<R, WAVE, NCW, VY>, &query_sweepx<R, WAVE, NCW, VY>, ST_T1_DEPTH};
  e.exch = 1;
  return e;
}

// ---- time-tiled heat sweep with every level in one warp's registers (sweeph.cuh, G5)
template <int R, int TK, int VY, int NW>
cudaError_t launch_sweeph(const KernelMaps& maps, const SweepParams& p, dim3 grid, int nslot,
                          size_t smem, cudaStream_t stream) {
  const int block = 32 * NW;
  const bool ev = p.wavelet != nullptr || p.trace != nullptr;   // sources / receivers in this run
  if (p.outS) {
    if (ev) return launch_pdl(sweeph_kernel<R, TK, VY, NW, 3>, grid, block, smem, stream, maps.u, p, nslot);
    return launch_pdl(sweeph_kernel<R, TK, VY, NW, 1>, grid, block, smem, stream, maps.u, p, nslot);
  }
  if (ev) return launch_pdl(sweeph_kernel<R, TK, VY, NW, 2>, grid, block, smem, stream, maps.u, p, nslot);
  return launch_pdl(sweeph_kernel<R, TK, VY, NW, 0>, grid, block, smem, stream, maps.u, p, nslot);
}

template <int R, int TK, int VY, int NW>
cudaError_t query_sweeph(size_t smem, cudaFuncAttributes* attr, int* bps, int nthreads) {
  auto k = sweeph_kernel<R, TK, VY, NW, 0>;
  cudaError_t e = cudaSuccess;
  for (auto kk : {k, sweeph_kernel<R, TK, VY, NW, 1>, sweeph_kernel<R, TK, VY, NW, 2>, sweeph_kernel<R, TK, VY, NW, 3>}) {
    e = cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (attr) {
    e = cudaFuncGetAttributes(attr, k);
    if (e != cudaSuccess) return e;
  }
  if (bps) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, nthreads, smem);
  return cudaSuccess;
}

#ifndef ST_TH_DEPTH
#define ST_TH_DEPTH 4   // heat time-tiled kernel: ring planes of prefetch beyond the radius+1 in use
#endif

template <int R, int TK, int VY, int NW>
constexpr KernelEntry make_entryH() {
  using G = GeomH<R, TK, VY, NW>;
  return KernelEntry{3, 1, R, TK, VY, NW, G::NTHREADS, G::OX, G::OY, G::BW, G::BH,
                     R, (size_t)G::SLOT_BYTES, (size_t)G::FIXED_BYTES,
                     &launch_sweeph<R, TK, VY, NW>, &query_sweeph<R, TK, VY, NW>, ST_TH_DEPTH};
}

}  // namespace st
