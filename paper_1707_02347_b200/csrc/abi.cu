// abi.cu -- plan, pass scheduling and the C ABI of libstencil.so (include/stencil.h).
//
// Host-side responsibilities:
//   * layout (a1): fp32 [Z][Y][X], X = round_up(nx,32), no x/y halo storage (TMA OOB zero fill
//     and in-kernel masks give the Dirichlet boundary), G = r*T_c ghost planes per z side for
//     z-slabs;
//   * medium precompute (a3): a, c per point once per run (kernel `medium_kernel`);
//   * pass schedule (a7, a8): nt steps = passes of T_k levels (time-tiled kernel, ping-pong
//     output pair) + single-level passes (in place), final swap/copy to honour the contract;
//   * z-slab bookkeeping (a9): shrinking valid plane ranges between halo exchanges;
//   * sources/receivers (a4, a5): filtered per slab, sorted by plane into per-plane tables.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/stencil.h"
#include "registry.h"
#include "resident.cuh"

namespace {

thread_local std::string g_err = "";

struct Buf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// NCCL, loaded at run time (the NCCL the process already has -- torch's libnccl.so.2 -- or
// $ST_NCCL_LIB), so libstencil.so has no link-time NCCL dependency.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  decltype(&ncclCommGetAsyncError) async_err = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* path = getenv("ST_NCCL_LIB");
    void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { a.why = std::string("dlopen NCCL failed: ") + dlerror(); return a; }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.get_id = reinterpret_cast<decltype(a.get_id)>(sym("ncclGetUniqueId"));
    a.init = reinterpret_cast<decltype(a.init)>(sym("ncclCommInitRank"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(sym("ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
    a.gstart = reinterpret_cast<decltype(a.gstart)>(sym("ncclGroupStart"));
    a.gend = reinterpret_cast<decltype(a.gend)>(sym("ncclGroupEnd"));
    a.allreduce = reinterpret_cast<decltype(a.allreduce)>(sym("ncclAllReduce"));
    a.errstr = reinterpret_cast<decltype(a.errstr)>(sym("ncclGetErrorString"));
    a.async_err = reinterpret_cast<decltype(a.async_err)>(sym("ncclCommGetAsyncError"));
    a.ok = a.get_id && a.init && a.destroy && a.send && a.recv && a.gstart && a.gend && a.allreduce &&
           a.errstr && a.async_err;
    if (!a.ok) a.why = "NCCL library lacks a required symbol";
    return a;
  }();
  return api;
}

}  // namespace

struct stencil_plan {
  st_config cfg{};
  std::vector<double> coeffs;
  cudaStream_t stream = nullptr;
  int device = 0;
  int sm_count = 148;
  // layout
  long long nx = 0, ny = 0, nzl = 0, X = 0, Y = 0, Z = 0, G = 0, z0g = 0;
  bool has_lo = false, has_hi = false;
  // kernels
  const st::KernelEntry* k_tk = nullptr;   // time-tiled (t_kernel) instance
  const st::KernelEntry* k_t1 = nullptr;   // single-level instance
  int nslot_tk = 0, nslot_t1 = 0;
  size_t smem_tk = 0, smem_t1 = 0;
  int bps_tk = 1, bps_t1 = 1;
  // coefficients
  float K0 = 0.f, W[3][st::kMaxR + 1] = {};
  float dtf = 0.f;
  // scratch
  Buf ac, p2, c2, tables;
  Buf a_pl, c_pl, aflag;               // planar medium + a == -1 tile flags (KernelEntry::askip)
  // two-role exchange passes (sweepx.cuh): tile table and u32 words [ticket, fault, prog[ntiles]]
  Buf xtiles, xwords, xtrace;
  std::vector<st::XTile> xx;           // host copy of the uploaded tile table
  int xt_lo = -1, xt_hi = -1;          // output plane range the table was built for
  int x_ntiles = 0;                    // tiles of that table
  unsigned x_ticket_base = 0, x_seq = 0;
  Buf staging;       // pinned host staging for the src/rec tables
  bool last_swapped = false;           // ST_NO_SWAP: the last run returned the pair swapped
  // fused halo push (stencil_set_peer)
  Buf counters;                        // 2 x u64 inbound push counters: [0] from lo, [1] from hi
  const float* my_ab[2] = {nullptr, nullptr};          // this rank's two field buffers
  float* peer_ab[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // [side][a/b] peer buffers
  unsigned long long* peer_ctr[2] = {nullptr, nullptr};              // neighbours' counters
  long long fused_runs = 0;            // fused runs issued since the peers were set
  std::vector<std::string> ipc_opened; // handles opened by stencil_ipc_open (released on destroy)
  // library-owned halo exchange (st_config.nccl_id): communicator, comm stream, join events
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  bool have_medium = false;            // a/c hold the medium of an earlier run (vel == NULL reuses it)
  bool have_tables = false;            // tables hold the src/rec lists below (re-uploaded on change)
  std::vector<int32_t> last_src, last_rec;
  const int *t_sb = nullptr, *t_rb = nullptr;
  const int4 *t_s = nullptr, *t_r = nullptr;
  cudaEvent_t staging_ev = nullptr;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  bool broken = false;
  mutable std::string err;             // also set by the const entry points (stencil_ipc_export)
  // timing (stencil_set_timing / stencil_timing)
  // one (start, end) event pair per timed run since the last stencil_timing query; the pool is
  // reused, so a run records events without any host synchronisation
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;   // 2 per pair
  int ev_used = 0;                    // pairs recorded since the last query
  int last_launches = 0, last_tiled = 0, last_aux = 0;   // accumulated since the last query
};

namespace {

st_status fail(const stencil_plan* p, st_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (p) p->err = buf;
  g_err = buf;
  return s;
}

st_status cuda_fail(stencil_plan* p, cudaError_t e, const char* what) {
  if (p && (e == cudaErrorIllegalAddress || e == cudaErrorLaunchFailure ||
            e == cudaErrorIllegalInstruction || e == cudaErrorMisalignedAddress))
    p->broken = true;
  return fail(p, ST_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CK(expr, what)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(p, _e, what); \
  } while (0)

long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

void free_buf(Buf& b) {
  if (b.ptr) cudaFree(b.ptr);
  b.ptr = nullptr;
  b.bytes = 0;
}

st_status ensure_buf(stencil_plan* p, Buf& b, size_t bytes, const char* what) {
  if (b.bytes >= bytes) return ST_OK;
  free_buf(b);
  cudaError_t e = cudaMalloc(&b.ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(p, ST_ENOMEM, "cudaMalloc(%zu) for %s failed: %s", bytes, what, cudaGetErrorString(e));
  }
  b.bytes = bytes;
  return ST_OK;
}

// ------------------------------------------------------------------ medium precompute (G0)
// Per point (fp32, denormals flushed, no contraction; P:1678-1708 rewritten, see stencil.h):
//   m = 1/(v*v); te = dt*eta; m2 = 2m; den = te + m2; a = (te - m2)/den; c = 2dt^2/den
__device__ __forceinline__ float mul_ftz(float a, float b) { float r; asm("mul.rn.ftz.f32 %0,%1,%2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float add_ftz(float a, float b) { float r; asm("add.rn.ftz.f32 %0,%1,%2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float sub_ftz(float a, float b) { float r; asm("sub.rn.ftz.f32 %0,%1,%2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float div_ftz(float a, float b) { float r; asm("div.rn.ftz.f32 %0,%1,%2;" : "=f"(r) : "f"(a), "f"(b)); return r; }

__device__ __forceinline__ void medium_point(float v, float eta, float dtf, float two_dt2, float& a, float& c) {
  const float m = div_ftz(1.0f, mul_ftz(v, v));
  const float te = mul_ftz(dtf, eta);
  const float m2 = mul_ftz(2.0f, m);
  const float den = add_ftz(te, m2);
  a = div_ftz(sub_ftz(te, m2), den);
  c = div_ftz(two_dt2, den);
}

// a_pl != nullptr (planar-medium kernels): a and c also as planar fp32 fields, and aflag (preset to
// 1) cleared for every (plane, oy-row x 64-column tile) holding an interior point with a != -1.
__global__ void medium_kernel(const float* __restrict__ vel, const float* __restrict__ damp,
                              float4* __restrict__ ac, int nx, int ny, long long X, long long plane,
                              int z_lo, int nplanes, float dtf, float two_dt2,
                              float* __restrict__ a_pl, float* __restrict__ c_pl,
                              unsigned char* __restrict__ aflag, int oy, int ntx, int nty) {
  const long long X2 = X >> 1;
  const long long per_plane = X2 * ny;
  const long long total = per_plane * nplanes;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long z = z_lo + i / per_plane;
    const long long rem = i % per_plane;
    const long long y = rem / X2;
    const long long xp = rem % X2;
    const long long x = 2 * xp;
    if (x >= nx) continue;
    const long long off = z * plane + y * X + x;
    const float2 v = *reinterpret_cast<const float2*>(vel + off);
    float2 e = make_float2(0.f, 0.f);
    if (damp) e = *reinterpret_cast<const float2*>(damp + off);
    float a0, c0, a1 = 0.f, c1 = 0.f;
    medium_point(v.x, e.x, dtf, two_dt2, a0, c0);
    if (x + 1 < nx) medium_point(v.y, e.y, dtf, two_dt2, a1, c1);
    ac[z * (plane >> 1) + y * X2 + xp] = make_float4(a0, a1, c0, c1);   // plane/2 float4 per plane
    if (a_pl) {
      *reinterpret_cast<float2*>(a_pl + off) = make_float2(a0, a1);
      *reinterpret_cast<float2*>(c_pl + off) = make_float2(c0, c1);
      if (!(a0 == -1.0f) || (x + 1 < nx && !(a1 == -1.0f)))
        aflag[(z * nty + y / oy) * ntx + (x >> 6)] = 0;
    }
  }
}

__global__ void swap_kernel(float4* __restrict__ a, float4* __restrict__ b, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 t = a[i];
    a[i] = b[i];
    b[i] = t;
  }
}

// ------------------------------------------------------------------ tensor maps
// 3-D fp32 map over the valid planes of a [Z][rows][row_elems]-strided array: dims (dim0, ny,
// valid planes), box (box_w, box_h, 1); out-of-bounds boxes are zero-filled (Dirichlet halo).
st_status encode_box(stencil_plan* p, const float* base, long long dim0, long long row_elems,
                     long long plane_elems, int box_w, int box_h, CUtensorMap* map) {
  const long long zv_lo = p->G - (p->has_lo ? p->G : 0);
  const long long zv_hi = p->G + p->nzl + (p->has_hi ? p->G : 0);
  void* b = const_cast<float*>(base + zv_lo * plane_elems);
  cuuint64_t dims[3] = {(cuuint64_t)dim0, (cuuint64_t)p->ny, (cuuint64_t)(zv_hi - zv_lo)};
  cuuint64_t strides[2] = {(cuuint64_t)(row_elems * 4), (cuuint64_t)(plane_elems * 4)};
  cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = p->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, b, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(p, ST_ECUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return ST_OK;
}

// u^n box with halo of instance k over a field
st_status encode_map(stencil_plan* p, const st::KernelEntry* k, const float* field, CUtensorMap* map) {
  return encode_box(p, field, p->nx, p->X, p->X * p->Y, k->bw, k->bh, map);
}

// choose ring depth / occupancy for one instance
st_status configure_instance(stencil_plan* p, const st::KernelEntry* k, int* nslot, size_t* smem, int* bps) {
  const size_t max_smem = 227 * 1024;
  const int min_slots = k->fixed_slots ? k->fixed_slots : k->rz + 2;
  const int want_slots = k->fixed_slots ? k->fixed_slots
                                        : std::min(64, k->rz + 1 + k->extra_depth);   // prefetch depth in planes
  int best_slots = 0, best_bps = 0;
  size_t best_smem = 0;
  for (int slots = std::max(min_slots, want_slots); slots >= min_slots; --slots) {
    const size_t sm = k->fixed_bytes + (size_t)slots * k->slot_bytes;
    if (sm > max_smem) continue;
    int b = 0;
    cudaError_t e = k->query(sm, nullptr, &b, k->nthreads);
    if (e != cudaSuccess) return cuda_fail(p, e, "occupancy query");
    if (b > best_bps || (b == best_bps && slots > best_slots)) {
      best_bps = b; best_slots = slots; best_smem = sm;
    }
  }
  if (best_slots == 0 || best_bps == 0)
    return fail(p, ST_EUNSUPPORTED, "kernel instance (R=%d, T_k=%d) does not fit on this device", k->radius, k->tk);
  // prefer two resident CTAs if a shallower ring allows it
  *nslot = best_slots; *smem = best_smem; *bps = best_bps;
  CK(k->query(best_smem, nullptr, nullptr, k->nthreads), "cudaFuncSetAttribute");
  return ST_OK;
}

// ------------------------------------------------------------------ source/receiver tables
struct Tables {
  int nsrc_local = 0, nrec_local = 0;
  size_t off_src_begin = 0, off_src = 0, off_rec_begin = 0, off_rec = 0, bytes = 0;
};

}  // namespace

extern "C" {

int32_t stencil_abi_version(void) { return 105; }

st_status stencil_nccl_unique_id(void* out) {
  if (!out) return fail(nullptr, ST_EINVAL, "out is NULL");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(nullptr, ST_ENCCL, "%s", api.why.c_str());
  ncclUniqueId id;
  const ncclResult_t r = api.get_id(&id);
  if (r != ncclSuccess) return fail(nullptr, ST_ENCCL, "ncclGetUniqueId: %s", api.errstr(r));
  memcpy(out, &id, sizeof id);
  return ST_OK;
}

#ifdef ST_XTRACE
// diagnostic builds only: copy the event trace of the last exchange pass and its tile table
int64_t stencil_xtrace(stencil_plan* p, void* host, int64_t bytes, void* tiles_host, int64_t tiles_bytes) {
  if (!p || !p->xtrace.ptr) return -1;
  cudaStreamSynchronize(p->stream);
  const size_t n = std::min<size_t>((size_t)bytes, p->xtrace.bytes);
  cudaMemcpy(host, p->xtrace.ptr, n, cudaMemcpyDeviceToHost);
  const size_t tn = std::min<size_t>((size_t)tiles_bytes, p->xx.size() * sizeof(st::XTile));
  memcpy(tiles_host, p->xx.data(), tn);
  return (int64_t)p->xx.size();
}
#endif

int32_t stencil_swapped(const stencil_plan* p) { return p ? (p->last_swapped ? 1 : 0) : -1; }

// ------------------------------------------------------------------ fused halo push (NEXT-1)
static bool fused_capable(const stencil_plan* p) {
  const st_config& c = p->cfg;
  return c.ndim == 3 && c.nranks > 1 && c.t_comm == 1 && c.t_kernel == 1;
}

static bool fused_ready(const stencil_plan* p) {
  return fused_capable(p) && p->my_ab[0] && (!p->has_lo || p->peer_ctr[0]) && (!p->has_hi || p->peer_ctr[1]);
}

st_status stencil_peer_counters(stencil_plan* p, unsigned long long** counters) {
  if (!p || !counters) return fail(p, ST_EINVAL, "plan or counters is NULL");
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  if (!p->counters.ptr) {
    st_status s = ensure_buf(p, p->counters, 2 * sizeof(unsigned long long), "push counters");
    if (s != ST_OK) return s;
    CK(cudaMemset(p->counters.ptr, 0, 2 * sizeof(unsigned long long)), "cudaMemset counters");
  }
  *counters = static_cast<unsigned long long*>(p->counters.ptr);
  return ST_OK;
}

st_status stencil_set_peer(stencil_plan* p, int32_t side, const float* my_a, const float* my_b,
                           float* peer_a, float* peer_b, unsigned long long* peer_counters) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  if (!fused_capable(p)) return fail(p, ST_EINVAL, "fused halo push needs ndim 3, nranks > 1, t_comm == t_kernel == 1");
  if (!(p->cfg.flags & ST_NO_SWAP))
    return fail(p, ST_EINVAL, "fused halo push needs a ST_NO_SWAP plan (a swap kernel would race with the peers' pushes)");
  if (side != 0 && side != 1) return fail(p, ST_EINVAL, "side must be 0 (lo) or 1 (hi)");
  if ((side == 0 && !p->has_lo) || (side == 1 && !p->has_hi)) return fail(p, ST_EINVAL, "rank has no neighbour on side %d", side);
  if (!my_a || !my_b || my_a == my_b || !peer_a || !peer_b || !peer_counters)
    return fail(p, ST_EINVAL, "null or aliased buffer / counter pointer");
  if (p->my_ab[0] && (p->my_ab[0] != my_a || p->my_ab[1] != my_b))
    return fail(p, ST_EINVAL, "my_a/my_b differ from the pair registered for the other side");
  unsigned long long* mine = nullptr;
  st_status s = stencil_peer_counters(p, &mine);       // make sure ours exist (the peer bumps them)
  if (s != ST_OK) return s;
  p->my_ab[0] = my_a; p->my_ab[1] = my_b;
  p->peer_ab[side][0] = peer_a; p->peer_ab[side][1] = peer_b;
  p->peer_ctr[side] = peer_counters;
  // the step count restarts: so does this side's inbound counter (no pushes may be in flight)
  CK(cudaMemsetAsync(mine + side, 0, sizeof(unsigned long long), p->stream), "cudaMemsetAsync counter");
  CK(cudaStreamSynchronize(p->stream), "cudaStreamSynchronize");
  p->fused_runs = 0;
  return ST_OK;
}

st_status stencil_ipc_export(const stencil_plan* p, const void* dev_ptr, void* blob) {
  if (!p || !dev_ptr || !blob) return fail(p, ST_EINVAL, "null argument");
  if (cudaSetDevice(p->device) != cudaSuccess) return fail(p, ST_ECUDA, "cudaSetDevice failed");
  // base of the allocation holding dev_ptr (torch's caching allocator sub-allocates segments)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return fail(p, ST_ECUDA, "cuMemGetAddressRange lookup failed");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn)(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return fail(p, ST_ECUDA, "cuMemGetAddressRange failed for %p", dev_ptr);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e != cudaSuccess) return fail(p, ST_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  const long long off = (long long)((CUdeviceptr)dev_ptr - base);
  memcpy(blob, &h, sizeof h);
  memcpy(static_cast<char*>(blob) + 64, &off, sizeof off);
  return ST_OK;
}

// One mapping per exported allocation and process: a second cudaIpcOpenMemHandle of a handle that
// is already open (two fields sub-allocated from one torch segment, or two plans with the same
// neighbour) is refused by the runtime, so opens are shared and reference-counted.
struct IpcMapping { void* base; int refs; };
static std::mutex g_ipc_mu;
static std::map<std::string, IpcMapping> g_ipc_open;

static void ipc_release(const std::string& key) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_open.find(key);
  if (it == g_ipc_open.end()) return;
  if (--it->second.refs == 0) {
    cudaIpcCloseMemHandle(it->second.base);
    g_ipc_open.erase(it);
  }
}

st_status stencil_ipc_open(stencil_plan* p, const void* blob, void** dev_ptr) {
  if (!p || !blob || !dev_ptr) return fail(p, ST_EINVAL, "null argument");
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  cudaIpcMemHandle_t h;
  long long off = 0;
  memcpy(&h, blob, sizeof h);
  memcpy(&off, static_cast<const char*>(blob) + 64, sizeof off);
  void* base = nullptr;
  const std::string key(static_cast<const char*>(blob), sizeof h);
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_open.find(key);
    if (it != g_ipc_open.end()) {
      it->second.refs++;
      base = it->second.base;
    } else {
      CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      g_ipc_open.emplace(key, IpcMapping{base, 1});
    }
  }
  p->ipc_opened.push_back(key);
  *dev_ptr = static_cast<char*>(base) + off;
  return ST_OK;
}

int32_t stencil_supported(int32_t ndim, int32_t time_order, int32_t radius, int32_t t_kernel) {
  return st::find_kernel(ndim, time_order, radius, t_kernel) != nullptr ? 1 : 0;
}

const char* stencil_last_error(const stencil_plan* p) {
  if (p) return p->err.c_str();
  return g_err.c_str();
}

st_status stencil_create(const st_config* cfg, stencil_plan** out) {
  stencil_plan* p = nullptr;
  if (!out) return fail(nullptr, ST_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, ST_EINVAL, "cfg is NULL");
  const st_config& c = *cfg;
  if (c.ndim != 2 && c.ndim != 3) return fail(nullptr, ST_EINVAL, "ndim must be 2 or 3 (got %d)", c.ndim);
  if (c.radius < 1 || c.radius > st::kMaxR) return fail(nullptr, ST_EINVAL, "radius must be in 1..%d (got %d)", st::kMaxR, c.radius);
  if (!c.coeffs) return fail(nullptr, ST_EINVAL, "coeffs is NULL");
  if (c.time_order != 1 && c.time_order != 2) return fail(nullptr, ST_EINVAL, "time_order must be 1 or 2");
  if (c.n[0] < 1 || c.n[1] < 1 || c.n[2] < 1) return fail(nullptr, ST_EINVAL, "grid sizes must be >= 1");
  if (c.ndim == 2 && c.n[2] != 1) return fail(nullptr, ST_EINVAL, "2-D problems need n[2] == 1");
  if (c.n[0] > (1ll << 30) || c.n[1] > (1ll << 30) || c.n[2] > (1ll << 30)) return fail(nullptr, ST_EINVAL, "grid too large");
  if (c.t_kernel < 1) return fail(nullptr, ST_EINVAL, "t_kernel must be >= 1");
  if (c.nranks < 1 || c.rank < 0 || c.rank >= c.nranks) return fail(nullptr, ST_EINVAL, "bad rank/nranks (%d/%d)", c.rank, c.nranks);
  if (c.nranks > 1 && c.ndim != 3) return fail(nullptr, ST_EINVAL, "z-slab decomposition needs ndim == 3");
  if (c.n[2] % c.nranks != 0) return fail(nullptr, ST_EINVAL, "n[2] %% nranks != 0");
  if (c.nranks > 1 && (c.t_comm < 1 || c.t_comm % c.t_kernel != 0)) return fail(nullptr, ST_EINVAL, "t_comm must be a positive multiple of t_kernel");
  if (c.nranks > 1 && (long long)c.radius * c.t_comm > c.n[2] / c.nranks)
    return fail(nullptr, ST_EINVAL, "ghost depth radius*t_comm (%lld) exceeds the slab thickness (%lld planes)",
                (long long)c.radius * c.t_comm, (long long)(c.n[2] / c.nranks));
  if (!(c.dt > 0) || !(c.dx[0] > 0) || !(c.dx[1] > 0) || (c.ndim == 3 && !(c.dx[2] > 0))) return fail(nullptr, ST_EINVAL, "dt and dx must be positive");
  if (!(c.flags & ST_FTZ)) return fail(nullptr, ST_EUNSUPPORTED, "only the flush-to-zero arithmetic mode is built (set ST_FTZ)");
  const st::KernelEntry* ktk = st::find_kernel(c.ndim, c.time_order, c.radius, c.t_kernel);
  const st::KernelEntry* kt1 = st::find_kernel(c.ndim, c.time_order, c.radius, 1);
  if (!ktk || !kt1) return fail(nullptr, ST_EUNSUPPORTED, "no compiled kernel for ndim=%d time_order=%d radius=%d t_kernel=%d", c.ndim, c.time_order, c.radius, c.t_kernel);

  p = new (std::nothrow) stencil_plan();
  if (!p) return fail(nullptr, ST_ENOMEM, "host allocation failed");
  p->cfg = c;
  p->coeffs.assign(c.coeffs, c.coeffs + c.radius + 1);
  p->cfg.coeffs = p->coeffs.data();
  p->stream = static_cast<cudaStream_t>(c.stream);
  p->device = c.device;
  p->k_tk = ktk;
  p->k_t1 = kt1;
  auto bail = [&](st_status s) { std::string m = g_err; stencil_destroy(p); g_err = m; return s; };

  cudaError_t e = cudaSetDevice(c.device);
  if (e != cudaSuccess) { cuda_fail(p, e, "cudaSetDevice"); return bail(ST_ECUDA); }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c.device);
  cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, c.device);
  if (major != 10) { fail(p, ST_EUNSUPPORTED, "device %d is not an sm_100 (Blackwell) GPU", c.device); return bail(ST_EUNSUPPORTED); }

  // layout
  p->nx = c.n[0]; p->ny = c.n[1];
  p->nzl = (c.ndim == 3) ? c.n[2] / c.nranks : 1;
  p->G = (c.nranks > 1) ? (long long)c.radius * c.t_comm : 0;
  p->X = round_up(p->nx, 32);
  p->Y = p->ny;
  p->Z = p->nzl + 2 * p->G;
  p->z0g = (long long)c.rank * p->nzl;
  p->has_lo = c.rank > 0;
  p->has_hi = c.rank < c.nranks - 1;

  // coefficients (double, axes summed x, y, z; see stencil.h)
  double k0 = 0.0;
  for (int a = 0; a < c.ndim; ++a) k0 += p->coeffs[0] / (c.dx[a] * c.dx[a]);
  p->K0 = (float)k0;
  for (int a = 0; a < c.ndim; ++a)
    for (int k = 1; k <= c.radius; ++k) p->W[a][k] = (float)(p->coeffs[k] / (c.dx[a] * c.dx[a]));
  p->dtf = (float)c.dt;

  // driver entry point for tensor-map encoding
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) { cuda_fail(p, e == cudaSuccess ? cudaErrorNotSupported : e, "cuTensorMapEncodeTiled lookup"); return bail(ST_ECUDA); }
  p->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);

  st_status s = configure_instance(p, ktk, &p->nslot_tk, &p->smem_tk, &p->bps_tk);
  if (s != ST_OK) return bail(s);
  s = configure_instance(p, kt1, &p->nslot_t1, &p->smem_t1, &p->bps_t1);
  if (s != ST_OK) return bail(s);

  // scratch: medium (wave), ping-pong pair (t_kernel > 1)
  const size_t field_bytes = (size_t)p->X * p->Y * p->Z * 4;
  if (c.time_order == 2) {
    s = ensure_buf(p, p->ac, 2 * field_bytes, "medium a/c");
    if (s != ST_OK) return bail(s);
    if (kt1->askip) {   // planar a, c and the a == -1 tile flags of the untiled static-ring kernel
      if (kt1->ox != 64) return bail(fail(p, ST_EUNSUPPORTED, "planar-medium kernel with a tile width other than 64"));
      s = ensure_buf(p, p->a_pl, field_bytes, "medium a (planar)");
      if (s == ST_OK) s = ensure_buf(p, p->c_pl, field_bytes, "medium c (planar)");
      if (s == ST_OK)
        s = ensure_buf(p, p->aflag, (size_t)p->Z * ((p->ny + kt1->oy - 1) / kt1->oy) * ((p->nx + 63) / 64), "a == -1 tile flags");
      if (s != ST_OK) return bail(s);
    }
  }
  if (c.t_kernel > 1) {
    s = ensure_buf(p, p->p2, field_bytes, "ping-pong u_prev");
    if (s == ST_OK) s = ensure_buf(p, p->c2, field_bytes, "ping-pong u_cur");
    if (s != ST_OK) return bail(s);
  }
  e = cudaEventCreateWithFlags(&p->staging_ev, cudaEventDisableTiming);
  if (e != cudaSuccess) { cuda_fail(p, e, "cudaEventCreate"); return bail(ST_ECUDA); }
  if (c.nccl_id) {
    // library-owned exchange: join the communicator (collective over the ranks; a one-rank plan
    // exercises the same time loop, comm stream and trace reduction with no neighbours)
    const NcclApi& api = nccl();
    if (!api.ok) { fail(p, ST_ENCCL, "%s", api.why.c_str()); return bail(ST_ENCCL); }
    ncclUniqueId id;
    memcpy(&id, c.nccl_id, sizeof id);
    const ncclResult_t r = api.init(&p->comm, c.nranks, id, c.rank);
    if (r != ncclSuccess) { p->comm = nullptr; fail(p, ST_ENCCL, "ncclCommInitRank: %s", api.errstr(r)); return bail(ST_ENCCL); }
    e = cudaStreamCreateWithFlags(&p->comm_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming);
    if (e != cudaSuccess) { cuda_fail(p, e, "comm stream/events"); return bail(ST_ECUDA); }
  }
  *out = p;
  return ST_OK;
}

st_status stencil_layout(const stencil_plan* p, int64_t padded[3], int64_t origin[3], int64_t zr[2]) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  if (padded) { padded[0] = p->X; padded[1] = p->Y; padded[2] = p->Z; }
  if (origin) { origin[0] = 0; origin[1] = 0; origin[2] = p->G; }
  if (zr) { zr[0] = p->z0g; zr[1] = p->z0g + p->nzl; }
  return ST_OK;
}

void stencil_destroy(stencil_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  free_buf(p->ac); free_buf(p->a_pl); free_buf(p->c_pl); free_buf(p->aflag); free_buf(p->p2); free_buf(p->c2); free_buf(p->tables);
  if (p->staging.ptr) cudaFreeHost(p->staging.ptr);
  if (p->staging_ev) cudaEventDestroy(p->staging_ev);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  for (const std::string& k : p->ipc_opened) ipc_release(k);
  free_buf(p->counters);
  free_buf(p->xtiles); free_buf(p->xwords); free_buf(p->xtrace);
  if (p->comm) { cudaStreamSynchronize(p->comm_stream); nccl().destroy(p->comm); }
  if (p->comm_stream) cudaStreamDestroy(p->comm_stream);
  if (p->ev_ready) cudaEventDestroy(p->ev_ready);
  if (p->ev_done) cudaEventDestroy(p->ev_done);
  delete p;
}

st_status stencil_set_timing(stencil_plan* p, int32_t enable) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  p->timing = enable != 0;
  p->ev_used = 0;
  p->last_launches = p->last_tiled = p->last_aux = 0;
  // pre-create event pairs so timed runs never call cudaEventCreate (a host cost that shows up
  // in the device time of launch-bound runs such as C1); the pool still grows if a caller runs
  // more than this many times between two queries
  while (p->timing && p->ev_pool.size() < 2 * 64) {
    cudaEvent_t e = nullptr;
    CK(cudaEventCreate(&e), "cudaEventCreate");
    p->ev_pool.push_back(e);
  }
  return ST_OK;
}

st_status stencil_timing(stencil_plan* p, float* ms, int32_t* launches, int32_t* tiled, int32_t* aux) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  if (!p->timing || p->ev_used == 0) return fail(p, ST_ESTATE, "no timed run (call stencil_set_timing first)");
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  CK(cudaEventSynchronize(p->ev_pool[2 * (p->ev_used - 1) + 1]), "timing event synchronize");
  float total = 0.f;
  for (int i = 0; i < p->ev_used; ++i) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, p->ev_pool[2 * i], p->ev_pool[2 * i + 1]), "cudaEventElapsedTime");
    total += t;
  }
  if (ms) *ms = total;
  if (launches) *launches = p->last_launches;
  if (tiled) *tiled = p->last_tiled;
  if (aux) *aux = p->last_aux;
  p->ev_used = 0;
  p->last_launches = p->last_tiled = p->last_aux = 0;
  return ST_OK;
}

st_status stencil_sync(stencil_plan* p) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  cudaSetDevice(p->device);
  cudaError_t e = cudaStreamSynchronize(p->stream);
  if (e != cudaSuccess) { p->broken = true; return cuda_fail(p, e, "stream synchronize"); }
  if (p->xwords.ptr) {   // an exchange pass whose wait timed out (sweepx.cuh)
    unsigned fault = 0;
    e = cudaMemcpy(&fault, static_cast<unsigned*>(p->xwords.ptr) + 1, sizeof fault, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { p->broken = true; return cuda_fail(p, e, "fault word read"); }
    if (fault) {
      p->broken = true;
      return fail(p, ST_ECUDA, "exchange pass: a tile's wait for the tiles it depends on timed out (results invalid)");
    }
  }
  return ST_OK;
}

static st_status upload_tables(stencil_plan* p, int32_t nsrc, const int32_t* src_xyz, int32_t nrec,
                               const int32_t* rec_xyz, const int** src_begin, const int4** src,
                               const int** rec_begin, const int4** rec) {
  // unchanged lists (the common case: every chunk of a simulation) -> the tables on the device
  // are still valid (they are only read by kernels, and any rewrite below is stream-ordered)
  if (p->have_tables && p->last_src.size() == (size_t)3 * nsrc && p->last_rec.size() == (size_t)3 * nrec &&
      (nsrc == 0 || memcmp(p->last_src.data(), src_xyz, 12 * (size_t)nsrc) == 0) &&
      (nrec == 0 || memcmp(p->last_rec.data(), rec_xyz, 12 * (size_t)nrec) == 0)) {
    *src_begin = p->t_sb; *src = p->t_s; *rec_begin = p->t_rb; *rec = p->t_r;
    return ST_OK;
  }
  p->have_tables = false;
  // sources: every plane of this slab's array (incl. ghosts) -> injected in redundant copies too
  // receivers: owned planes only (unique writer per slab)
  std::vector<int4> S, Rv;
  const long long zlo_arr = p->G - (p->has_lo ? p->G : 0), zhi_arr = p->G + p->nzl + (p->has_hi ? p->G : 0);
  for (int i = 0; i < nsrc; ++i) {
    const long long z = (p->cfg.ndim == 3) ? src_xyz[3 * i + 2] - p->z0g + p->G : 0;
    if (z >= zlo_arr && z < zhi_arr) S.push_back(make_int4(src_xyz[3 * i], src_xyz[3 * i + 1], (int)z, i));
  }
  for (int i = 0; i < nrec; ++i) {
    const long long z = (p->cfg.ndim == 3) ? rec_xyz[3 * i + 2] - p->z0g + p->G : 0;
    if (z >= p->G && z < p->G + p->nzl) Rv.push_back(make_int4(rec_xyz[3 * i], rec_xyz[3 * i + 1], (int)z, i));
  }
  auto by_plane = [](const int4& a, const int4& b) { return a.z < b.z; };
  std::stable_sort(S.begin(), S.end(), by_plane);    // stable: index order within a point
  std::stable_sort(Rv.begin(), Rv.end(), by_plane);
  const int Zp1 = (int)p->Z + 1;
  std::vector<int> sb(Zp1, 0), rb(Zp1, 0);
  {
    size_t i = 0;
    for (int z = 0; z < Zp1; ++z) { while (i < S.size() && S[i].z < z) ++i; sb[z] = (int)i; }
    i = 0;
    for (int z = 0; z < Zp1; ++z) { while (i < Rv.size() && Rv[i].z < z) ++i; rb[z] = (int)i; }
  }
  const size_t b_sb = Zp1 * sizeof(int), b_s = std::max<size_t>(1, S.size()) * sizeof(int4);
  const size_t b_rb = Zp1 * sizeof(int), b_r = std::max<size_t>(1, Rv.size()) * sizeof(int4);
  const size_t o_s = round_up(b_sb, 16), o_rb = o_s + round_up(b_s, 16), o_r = o_rb + round_up(b_rb, 16);
  const size_t total = o_r + b_r;
  st_status s = ensure_buf(p, p->tables, total, "source/receiver tables");
  if (s != ST_OK) return s;
  if (p->staging.bytes < total) {
    if (p->staging.ptr) { cudaEventSynchronize(p->staging_ev); cudaFreeHost(p->staging.ptr); }
    p->staging.ptr = nullptr; p->staging.bytes = 0;
    CK(cudaMallocHost(&p->staging.ptr, total), "cudaMallocHost");
    p->staging.bytes = total;
  } else {
    CK(cudaEventSynchronize(p->staging_ev), "staging event");
  }
  char* h = static_cast<char*>(p->staging.ptr);
  memcpy(h, sb.data(), b_sb);
  if (!S.empty()) memcpy(h + o_s, S.data(), S.size() * sizeof(int4));
  memcpy(h + o_rb, rb.data(), b_rb);
  if (!Rv.empty()) memcpy(h + o_r, Rv.data(), Rv.size() * sizeof(int4));
  CK(cudaMemcpyAsync(p->tables.ptr, h, total, cudaMemcpyHostToDevice, p->stream), "table upload");
  CK(cudaEventRecord(p->staging_ev, p->stream), "staging event record");
  char* d = static_cast<char*>(p->tables.ptr);
  *src_begin = reinterpret_cast<const int*>(d);
  *src = reinterpret_cast<const int4*>(d + o_s);
  *rec_begin = reinterpret_cast<const int*>(d + o_rb);
  *rec = reinterpret_cast<const int4*>(d + o_r);
  p->t_sb = *src_begin; p->t_s = *src; p->t_rb = *rec_begin; p->t_r = *rec;
  p->last_src.assign(src_xyz, src_xyz + 3 * (size_t)nsrc);
  p->last_rec.assign(rec_xyz, rec_xyz + 3 * (size_t)nrec);
  p->have_tables = true;
  return ST_OK;
}

static int choose_chunks(const stencil_plan* p, const st::KernelEntry* k, int bps, long long tiles, long long planes) {
  if (const char* e = getenv("ST_CHUNKS")) return std::max(1, atoi(e));   // tuning override
  const long long slots = (long long)p->sm_count * std::max(1, bps);
  double best = 1e300;
  int bestc = 1;
  for (int c = 1; c <= 32; ++c) {
    const long long chunk = (planes + c - 1) / c;
    if (c > 1 && chunk < 8) break;
    const long long ctas = tiles * c;
    const long long waves = (ctas + slots - 1) / slots;
    const double per = (double)chunk + 2.0 * k->rz * k->tk;   // warm-up + redundant levels
    const double t = waves * per;
    if (t < best * 0.999) { best = t; bestc = c; }
  }
  // static-ring instances (r = 5, 6, 8) measured faster with >= ~16 waves of shorter chunks than
  // the model above predicts (C5: 3 chunks 273.5, 6 chunks 280.1-280.6, 8 chunks 281.4-281.7
  // GPts/s, same box; C4 unchanged at 2-4 chunks): split further while chunks stay >= 8r planes
  if (k->fixed_slots > 0 && k->tk == 1) {
    while (bestc < 32 && (tiles * bestc + slots - 1) / slots < 16 &&
           (planes + bestc) / (bestc + 1) >= 8LL * k->rz)
      ++bestc;
  }
  return bestc;
}

// ------------------------------------------------------------------ two-role exchange pass plan
// Tiles of one sweepx pass (sweepx.cuh header): L1 tiles on the regular 64 x H grid, L2 tiles on
// the same grid shifted r rows up, in the ticket order L1 row 0, L2 row 0, L1 row 1, ... per
// z-chunk; an L2 tile waits on the L1 tiles of its own and the previous row and the x-neighbours.
static void plan_xtiles(const stencil_plan* p, const st::KernelEntry* k, int out_lo, int out_hi,
                        int slots, std::vector<st::XTile>& T) {
  const int H = k->oy, r = k->radius;
  const int nx = (int)p->nx, ny = (int)p->ny;
  const int tx = (nx + 63) / 64;
  const int rows1 = (ny + H - 1) / H;            // L1 rows [jH, jH+H)
  const int rows2 = (ny + r + H - 1) / H;        // L2 rows [jH-r, jH+H-r)
  const int zv_lo = (int)(p->G - (p->has_lo ? p->G : 0));
  const int zv_hi = (int)(p->G + p->nzl + (p->has_hi ? p->G : 0));
  const long long planes = out_hi - out_lo;
  int best_c = 1;
  double best_t = 1e300;
  const long long per_chunk = (long long)tx * (rows1 + rows2);
  for (int c = 1; c <= 32; ++c) {
    const long long chunk = (planes + c - 1) / c;
    if (c > 1 && chunk < std::max(8, 2 * r)) break;
    const long long ntile = c * per_chunk;
    // waves x (chunk planes + the 2r-plane warm-up + the r-plane L1 overlap on each side)
    const double t = (double)((ntile + slots - 1) / slots) * (double)(chunk + 3 * r);
    if (t < best_t * 0.999) { best_t = t; best_c = c; }
  }
  if (const char* e = getenv("ST_EXCH_CHUNKS")) best_c = std::max(1, std::min<int>(atoi(e), (int)planes));
  const int zc = (int)((planes + best_c - 1) / best_c);
  T.clear();
  for (int c = 0; c < best_c; ++c) {
    const int czb = out_lo + c * zc, cze = std::min(out_hi, czb + zc);
    if (czb >= cze) break;
    const int base = (int)T.size();
    std::vector<int> l1_index((size_t)rows1 * tx, -1);
    std::vector<int> l2_index((size_t)rows2 * tx, -1);
    for (int j = 0; j < std::max(rows1, rows2); ++j) {
      if (j < rows1) {
        for (int i = 0; i < tx; ++i) {
          st::XTile d{};
          d.x0 = 64 * i; d.y0 = j * H; d.role = 0;
          d.zb = std::max(czb - r, zv_lo); d.ze = std::min(cze + r, zv_hi);
          d.oz0 = czb; d.oz1 = cze;
          d.nd = 0;
          d.partner = -1;
          for (int q = 0; q < 9; ++q) d.dep[q] = -1;
          l1_index[(size_t)j * tx + i] = (int)T.size();
          T.push_back(d);
        }
      }
      if (j < rows2) {
        for (int i = 0; i < tx; ++i) {
          st::XTile d{};
          d.x0 = 64 * i; d.y0 = j * H - r; d.role = 1;
          d.zb = czb; d.ze = cze; d.oz0 = czb; d.oz1 = cze;
          for (int q = 0; q < 9; ++q) d.dep[q] = -1;
          // the u^{n+1} box covers rows [jH-2r, jH+H) and columns [64i-r, 64i+64+r)
          const int ylo = std::max(0, j * H - 2 * r), yhi = std::min(ny, j * H + H);
          int nd = 0;
          if (ylo < yhi) {
            for (int jj = ylo / H; jj <= (yhi - 1) / H && jj < rows1; ++jj)
              for (int ii = std::max(0, i - 1); ii <= std::min(tx - 1, i + 1); ++ii)
                if (nd < 9) d.dep[nd++] = l1_index[(size_t)jj * tx + ii];
          }
          d.nd = nd;
          d.partner = -1;
          l2_index[(size_t)j * tx + i] = (int)T.size();
          if (j < rows1) T[(size_t)l1_index[(size_t)j * tx + i]].partner = (int)T.size();
          T.push_back(d);
        }
      }
    }
    (void)base;
  }
}

// ------------------------------------------------------------------ resident 2-D run (G4)
extern "C++" {
typedef void (*res_kernel_t)(const st::SweepParams, float*, float*, const float*, const float*, int, int);
template <int R>
static res_kernel_t res_pick(bool wave) {
  return wave ? &st::resident2d_kernel<R, true> : &st::resident2d_kernel<R, false>;
}
static res_kernel_t res_kernel(int R, bool wave) {
  switch (R) {
    case 1: return res_pick<1>(wave); case 2: return res_pick<2>(wave);
    case 3: return res_pick<3>(wave); case 4: return res_pick<4>(wave);
    case 5: return res_pick<5>(wave); case 6: return res_pick<6>(wave);
    case 7: return res_pick<7>(wave); default: return res_pick<8>(wave);
  }
}
// whole run of a 2-D plan in one CTA when both time levels (+ medium) fit in shared memory
static bool res_fits(const stencil_plan* p) {
  if (p->cfg.ndim != 2 || p->cfg.nranks != 1) return false;
  if (getenv("ST_NO_RESIDENT")) return false;   // test/measurement override: per-step sweeps
  for (int cap : {st::RES_CLUSTER, 8}) {   // the launch may fall back to 8-CTA clusters
    const int cs = st::res_cluster(p->cfg.radius, (int)p->ny, cap);
    const int spb = st::res_spb(p->cfg.radius, (int)p->ny, cs);
    if (st::res_smem_bytes(p->cfg.radius, p->cfg.time_order == 2, (int)p->nx, (int)p->ny, cs, spb) > 227 * 1024)
      return false;
  }
  return true;
}
}  // extern "C++"

// zr_lo/zr_hi >= 0 (internal, nt == 1, T = 1): sweep only the output planes [zr_lo, zr_hi)
// (the boundary bands / interior split of the overlapped exchange).  internal: the library-owned
// exchange drives this call -- no nt <= t_comm check, and the pair is left swapped (reported in
// p->last_swapped) instead of restored.
static st_status run_impl(stencil_plan* p, float* u_prev, float* u_cur, const float* vel,
                          const float* damp, int32_t nt, int64_t step0, int32_t nsrc,
                          const int32_t* src_xyz, const float* src_wavelet, int32_t nrec,
                          const int32_t* rec_xyz, float* rec_trace, int32_t save_every,
                          float* snapshots, int64_t snap_stride, int zr_lo = -1, int zr_hi = -1,
                          bool internal = false, const float* in_prev = nullptr,
                          const float* in_cur = nullptr) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  if (p->broken) return fail(p, ST_ESTATE, "plan is in an error state after an earlier CUDA fault");
  const st_config& c = p->cfg;
  const bool wave = c.time_order == 2;
  if (!u_prev || !u_cur) return fail(p, ST_EINVAL, "u_prev/u_cur is NULL");
  if (u_prev == u_cur) return fail(p, ST_EINVAL, "u_prev and u_cur must be distinct buffers");
  if (wave && !vel && !p->have_medium)
    return fail(p, ST_ESTATE, "vel is NULL but no earlier run of this plan computed the medium");
  if (nt < 0) return fail(p, ST_EINVAL, "nt < 0");
  if (step0 < 0) return fail(p, ST_EINVAL, "step0 < 0");
  if (nsrc < 0 || nrec < 0) return fail(p, ST_EINVAL, "negative source/receiver count");
  if (nsrc > 0 && (!src_xyz || !src_wavelet)) return fail(p, ST_EINVAL, "sources need src_xyz and src_wavelet");
  if (nrec > 0 && (!rec_xyz || !rec_trace)) return fail(p, ST_EINVAL, "receivers need rec_xyz and rec_trace");
  if (c.nranks > 1 && nt > c.t_comm && !internal)
    return fail(p, ST_EINVAL, "nt (%d) > t_comm (%d) with nranks > 1", nt, c.t_comm);
  if (zr_lo >= 0 && (nt != 1 || c.t_kernel != 1 || zr_hi <= zr_lo)) return fail(p, ST_EINVAL, "plane-range sweep needs nt == 1, t_kernel == 1");
  const long long nzg = c.n[2];
  for (int i = 0; i < nsrc; ++i) {
    const int32_t* q = src_xyz + 3 * i;
    if (q[0] < 0 || q[0] >= c.n[0] || q[1] < 0 || q[1] >= c.n[1] || q[2] < 0 || q[2] >= nzg)
      return fail(p, ST_EINVAL, "source %d (%d,%d,%d) outside the interior", i, q[0], q[1], q[2]);
  }
  for (int i = 0; i < nrec; ++i) {
    const int32_t* q = rec_xyz + 3 * i;
    if (q[0] < 0 || q[0] >= c.n[0] || q[1] < 0 || q[1] >= c.n[1] || q[2] < 0 || q[2] >= nzg)
      return fail(p, ST_EINVAL, "receiver %d (%d,%d,%d) outside the interior", i, q[0], q[1], q[2]);
  }
  if (nt == 0) return ST_OK;
  // fused halo push: every run is one T = 1 pass whose output field is one of the registered pair
  const bool fused = fused_ready(p);
  if (fused && u_prev != p->my_ab[0] && u_prev != p->my_ab[1])
    return fail(p, ST_EINVAL, "fused halo push: u_prev is neither of the buffers given to stencil_set_peer");
  if (fused && save_every > 0) return fail(p, ST_EINVAL, "fused halo push does not combine with snapshots");
  int aux_launches = 0;
  CK(cudaSetDevice(p->device), "cudaSetDevice");

  const long long zv_lo = p->G - (p->has_lo ? p->G : 0);
  const long long zv_hi = p->G + p->nzl + (p->has_hi ? p->G : 0);
  const long long plane = p->X * p->Y;

  // medium a/c over all valid planes (vel == NULL: keep the medium of the previous run, e.g. the
  // later T_c-step chunks of one z-slab simulation)
  if (wave && vel) {
    const long long n = (p->X / 2) * p->Y * (zv_hi - zv_lo);
    const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)p->sm_count * 16);
    const bool planar = p->k_t1->askip != 0;
    const int fl_oy = p->k_t1->oy, fl_ntx = (int)((p->nx + 63) / 64), fl_nty = (int)((p->ny + fl_oy - 1) / fl_oy);
    if (planar)
      CK(cudaMemsetAsync(p->aflag.ptr, 1, (size_t)p->Z * fl_nty * fl_ntx, p->stream), "aflag reset");
    medium_kernel<<<blocks, 256, 0, p->stream>>>(vel, damp, static_cast<float4*>(p->ac.ptr), (int)p->nx, (int)p->ny,
                                                  p->X, plane, (int)zv_lo, (int)(zv_hi - zv_lo), p->dtf,
                                                  (float)(2.0 * c.dt * c.dt),
                                                  planar ? static_cast<float*>(p->a_pl.ptr) : nullptr,
                                                  planar ? static_cast<float*>(p->c_pl.ptr) : nullptr,
                                                  planar ? static_cast<unsigned char*>(p->aflag.ptr) : nullptr,
                                                  fl_oy, fl_ntx, fl_nty);
    CK(cudaGetLastError(), "medium kernel launch");
    p->have_medium = true;
    ++aux_launches;
  }

  const int *sbeg, *rbeg;
  const int4 *sarr, *rarr;
  st_status s = upload_tables(p, nsrc, src_xyz, nrec, rec_xyz, &sbeg, &sarr, &rbeg, &rarr);
  if (s != ST_OK) return s;

  // buffers: 0 = caller P, 1 = caller C, 2 = scratch P2, 3 = scratch C2
  float* bufs[4] = {u_prev, u_cur, static_cast<float*>(p->p2.ptr), static_cast<float*>(p->c2.ptr)};
  int prev = 0, cur = 1;
  CUtensorMap maps_t1[4], maps_tk[4], maps_p0[4], maps_u1[4], maps_l1[4], map_a0, map_a1, map_c_pl, map_a_pl;
  bool have_t1[4] = {false, false, false, false}, have_tk[4] = {false, false, false, false};
  bool have_l1[4] = {false, false, false, false};
  bool have_p0[4] = {false, false, false, false}, have_u1[4] = {false, false, false, false};
  bool have_ac = false, have_pl = false;
  st::KernelMaps km{};

  st::SweepParams sp{};
  sp.nx = (int)p->nx; sp.ny = (int)p->ny; sp.X = (int)p->X; sp.plane = plane;
  sp.gz_lo = p->has_lo ? 0 : (int)p->G;
  sp.gz_hi = p->has_hi ? (int)p->Z : (int)(p->G + p->nzl);
  sp.zv_lo = (int)zv_lo;
  sp.zv_hi = (int)zv_hi;
  sp.ac = static_cast<const float4*>(p->ac.ptr);
  sp.aflag = static_cast<const unsigned char*>(p->aflag.ptr);
  sp.fl_ntx = (int)((p->nx + 63) / 64);
  sp.fl_nty = (int)((p->ny + p->k_t1->oy - 1) / p->k_t1->oy);
  sp.K0 = p->K0; sp.dt = p->dtf;
  memcpy(sp.W, p->W, sizeof sp.W);
  sp.iso = 1;
  for (int k = 1; k <= c.radius; ++k)
    for (int a = 1; a < c.ndim; ++a)
      if (memcmp(&p->W[a][k], &p->W[0][k], sizeof(float)) != 0) sp.iso = 0;
  sp.src_begin = sbeg; sp.src = sarr; sp.wavelet = src_wavelet; sp.wl_stride = nsrc;
  sp.rec_begin = rbeg; sp.rec = rarr; sp.trace = rec_trace; sp.tr_stride = nrec;

  int j = 0;
  int launches = 0, tiled_launches = 0;
  const bool resident = save_every <= 0 && !fused && zr_lo < 0 && res_fits(p);
  // stencil_run_from hands the initial pair here only for runs the resident kernel serves
  if (in_cur && !resident) return fail(p, ST_EINVAL, "internal: initial pair without a resident run");
  cudaEvent_t t_ev1 = nullptr;
  if (p->timing) {
    if ((int)p->ev_pool.size() < 2 * (p->ev_used + 1)) {
      // grows by one pair per run between two queries (the caller's query cadence bounds it)
      cudaEvent_t a = nullptr, b = nullptr;
      CK(cudaEventCreate(&a), "cudaEventCreate");
      CK(cudaEventCreate(&b), "cudaEventCreate");
      p->ev_pool.push_back(a); p->ev_pool.push_back(b);
    }
    CK(cudaEventRecord(p->ev_pool[2 * p->ev_used], p->stream), "timing event");
    t_ev1 = p->ev_pool[2 * p->ev_used + 1];
  }
  if (resident) {
    // G4: all nt steps in shared memory, one launch; the kernel writes (u^{n+nt-1}, u^{n+nt})
    // straight into (u_prev, u_cur)
    sp.wl_step = step0;
    sp.tr_step = 0;
    sp.out_lo = (int)p->G; sp.out_hi = (int)(p->G + p->nzl);
    // 16-CTA clusters (non-portable) measured faster than 8 on C1 (50.6 vs 60.7 us per 80
    // steps); fall back to the portable 8 if the device refuses the larger cluster
    cudaError_t le = cudaErrorUnknown;
    for (int cap : {st::RES_CLUSTER, 8}) {
      const int cs = st::res_cluster(c.radius, (int)p->ny, cap);
      int spb = st::res_spb(c.radius, (int)p->ny, cs);
      if (const char* e = getenv("ST_RES_SPB")) spb = std::max(1, std::min(spb, atoi(e)));   // tests
      const size_t smem = st::res_smem_bytes(c.radius, wave, (int)p->nx, (int)p->ny, cs, spb);
      res_kernel_t kf = res_kernel(c.radius, wave);
      CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "resident smem");
      if (cs > 8 && cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3((unsigned)cs);
      lc.blockDim = dim3(st::RES_THREADS);
      lc.dynamicSmemBytes = smem;
      lc.stream = p->stream;
      cudaLaunchAttribute la[2];
      la[0].id = cudaLaunchAttributeClusterDimension;
      la[0].val.clusterDim.x = (unsigned)cs; la[0].val.clusterDim.y = 1; la[0].val.clusterDim.z = 1;
      la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      la[1].val.programmaticStreamSerializationAllowed = ST_PDL;
      lc.attrs = la;
      lc.numAttrs = 2;
      le = cudaLaunchKernelEx(&lc, kf, sp, u_prev, u_cur, (const float*)(in_cur ? in_prev : u_prev),
                              (const float*)(in_cur ? in_cur : u_cur), (int)nt, spb);
      if (le == cudaSuccess) break;
      cudaGetLastError();
      if (cap == 8) break;
    }
    CK(le, "resident kernel launch");
    ++launches;
    tiled_launches += 1;
    j = nt;
  }
  while (j < nt) {
    // a time-tiled pass never crosses a snapshot step (passes end on multiples of save_every)
    const bool tiled = (c.t_kernel > 1) && (nt - j >= c.t_kernel) &&
                       (save_every <= 0 || (j % save_every) + c.t_kernel <= save_every);
    const int steps = tiled ? c.t_kernel : 1;
    const st::KernelEntry* k = tiled ? p->k_tk : p->k_t1;
    const int nslot = tiled ? p->nslot_tk : p->nslot_t1;
    const size_t smem = tiled ? p->smem_tk : p->smem_t1;
    const int bps = tiled ? p->bps_tk : p->bps_t1;
    CUtensorMap* maps = tiled ? maps_tk : maps_t1;
    bool* have = tiled ? have_tk : have_t1;
    if (!have[cur]) {
      s = encode_map(p, k, bufs[cur], &maps[cur]);
      if (s != ST_OK) return s;
      have[cur] = true;
    }
    km.u = maps[cur];
    if (k->ebw > 0) {   // producer-streamed u^{n-1}, u^n and medium boxes (time-tiled wave)
      if (!have_ac) {
        const float* acf = static_cast<const float*>(p->ac.ptr);
        s = encode_box(p, acf, 2 * p->X, 2 * p->X, 2 * plane, 128, k->eh0, &map_a0);
        if (s == ST_OK) s = encode_box(p, acf, 2 * p->X, 2 * p->X, 2 * plane, 128, k->eh1, &map_a1);
        if (s != ST_OK) return s;
        have_ac = true;
      }
      if (!have_p0[prev]) {
        s = encode_box(p, bufs[prev], p->nx, p->X, plane, k->ebw, k->eh0, &maps_p0[prev]);
        if (s != ST_OK) return s;
        have_p0[prev] = true;
      }
      if (!have_u1[cur]) {
        s = encode_box(p, bufs[cur], p->nx, p->X, plane, k->ebw, k->eh1, &maps_u1[cur]);
        if (s != ST_OK) return s;
        have_u1[cur] = true;
      }
      km.p0 = maps_p0[prev]; km.a0 = map_a0; km.u1 = maps_u1[cur]; km.a1 = map_a1;
      if (k->askip) {   // planar medium: a0 = c box, a1 = a box (same geometry as the u^{n-1} box)
        if (!have_pl) {
          s = encode_box(p, static_cast<const float*>(p->c_pl.ptr), p->nx, p->X, plane, k->ebw, k->eh0, &map_c_pl);
          if (s == ST_OK)
            s = encode_box(p, static_cast<const float*>(p->a_pl.ptr), p->nx, p->X, plane, k->ebw, k->eh0, &map_a_pl);
          if (s != ST_OK) return s;
          have_pl = true;
        }
        km.a0 = map_c_pl; km.a1 = map_a_pl;
      }
    }
    // output plane range after j+steps of the nt steps covered by the ghost zones
    const long long shrink = (long long)(nt - j - steps) * c.radius;
    sp.out_lo = (int)(p->has_lo ? p->G - shrink : p->G);
    sp.out_hi = (int)(p->has_hi ? p->G + p->nzl + shrink : p->G + p->nzl);
    if (zr_lo >= 0) { sp.out_lo = zr_lo; sp.out_hi = zr_hi; }
    sp.P = bufs[prev];
    sp.C = bufs[cur];
    int new_prev, new_cur;
    if (!tiled) {
      sp.outP = bufs[prev];            // in place: u^{n+1} over u^{n-1}
      sp.outC = nullptr;
      new_prev = cur; new_cur = prev;
    } else {
      const bool in_caller = prev < 2;
      const int op = in_caller ? 2 : 0, oc = in_caller ? 3 : 1;
      sp.outP = bufs[op];
      sp.outC = bufs[oc];
      new_prev = op; new_cur = oc;
    }
    sp.write_prev = (j + steps == nt) ? 1 : 0;
    sp.outS = (save_every > 0 && (j + steps) % save_every == 0)
                  ? snapshots + (long long)((j + steps) / save_every - 1) * snap_stride
                  : nullptr;
    sp.wl_step = step0 + j;
    sp.tr_step = j;
    const long long tiles = ((p->nx + k->ox - 1) / k->ox) * ((p->ny + k->oy - 1) / k->oy);
    const long long planes = sp.out_hi - sp.out_lo;
    const int chunks = choose_chunks(p, k, bps, tiles, planes);
    sp.zchunk = (int)((planes + chunks - 1) / chunks);
    dim3 grid((unsigned)((p->nx + k->ox - 1) / k->ox), (unsigned)((p->ny + k->oy - 1) / k->oy), (unsigned)chunks);
    sp.x_tiles = nullptr; sp.x_ntiles = 0; sp.x_ticket = sp.x_prog = sp.x_fault = nullptr;
    sp.x_trace = nullptr;
    if (k->exch) {
      // exchange-tiled pass: tile table (rebuilt when the output plane range changes), ticket,
      // progress words; level-1 box map over this pass's u^{n+1} output field
      if (p->xt_lo != sp.out_lo || p->xt_hi != sp.out_hi) {
        plan_xtiles(p, k, sp.out_lo, sp.out_hi, p->sm_count * std::max(1, bps), p->xx);
        const size_t tb = p->xx.size() * sizeof(st::XTile), nt_ = p->xx.size();
        const void* hsrc = p->xx.data();
        p->x_ntiles = (int)nt_;
        s = ensure_buf(p, p->xtiles, tb, "tile table");
        if (s != ST_OK) return s;
        CK(cudaMemcpyAsync(p->xtiles.ptr, hsrc, tb, cudaMemcpyHostToDevice, p->stream), "tile table upload");
        // a new table restarts the ticket and progress sequence (words zeroed, stream-ordered
        // after every earlier pass): progress values are base + plane with base = seq << 16, so a
        // word is "older than this launch" iff (int)(word - base) < 0
        const size_t wb = (2 + nt_) * sizeof(unsigned);
        s = ensure_buf(p, p->xwords, wb, "exchange words");
        if (s != ST_OK) return s;
        CK(cudaMemsetAsync(p->xwords.ptr, 0, wb, p->stream), "exchange words reset");
        p->x_ticket_base = 0;
        p->x_seq = 1;
        p->xt_lo = sp.out_lo; p->xt_hi = sp.out_hi;
      }
      const int op = (sp.outP == bufs[0]) ? 0 : (sp.outP == bufs[1]) ? 1 : (sp.outP == bufs[2]) ? 2 : 3;
      if (!have_l1[op]) {
        s = encode_map(p, k, bufs[op], &maps_l1[op]);
        if (s != ST_OK) return s;
        have_l1[op] = true;
      }
      km.u1 = maps_l1[op];
      unsigned* w = static_cast<unsigned*>(p->xwords.ptr);
      sp.x_tiles = p->xtiles.ptr;
      sp.x_ntiles = p->x_ntiles;
      sp.x_ticket = w;
      sp.x_fault = w + 1;
      sp.x_prog = w + 2;
      sp.x_ticket_base = p->x_ticket_base;
      sp.x_prog_base = p->x_seq << 16;
      sp.x_trace = nullptr;
#ifdef ST_XTRACE
      {
        const size_t tb = (size_t)p->x_ntiles * (size_t)ST_XTRACE_K * 12 * 8;
        s = ensure_buf(p, p->xtrace, tb, "trace");
        if (s != ST_OK) return s;
        CK(cudaMemsetAsync(p->xtrace.ptr, 0, tb, p->stream), "trace reset");
        sp.x_trace = static_cast<unsigned long long*>(p->xtrace.ptr);
      }
#endif
      p->x_ticket_base += (unsigned)p->x_ntiles;
      if (++p->x_seq == 0x8000u) {   // keep base < 2^31: restart the sequence (words zeroed)
        CK(cudaMemsetAsync(p->xwords.ptr, 0, (2 + (size_t)p->x_ntiles) * sizeof(unsigned), p->stream), "exchange words reset");
        p->x_ticket_base = 0;
        p->x_seq = 1;
      }
      grid = dim3((unsigned)p->x_ntiles, 1, 1);
    }
    sp.push_lo = sp.push_hi = nullptr;
    sp.band_lo = INT_MIN; sp.band_hi = INT_MAX;
    sp.sig_lo = sp.sig_hi = nullptr;
    sp.wait_lo = sp.wait_hi = nullptr;
    sp.wait_lo_target = sp.wait_hi_target = 0;
    if (fused) {
      // the band planes of u^{n+1} go straight into the neighbours' ghost zones (their output
      // field of this step, which corresponds to ours: the ranks advance in lockstep)
      const int ob = (sp.outP == p->my_ab[0]) ? 0 : 1;
      const int r = c.radius;
      // CTAs whose chunk produces band planes (identical geometry on every rank)
      long long n_lo = 0, n_hi = 0;
      for (int ch = 0; ch < chunks; ++ch) {
        const long long zb = sp.out_lo + (long long)ch * sp.zchunk, ze = std::min<long long>(sp.out_hi, zb + sp.zchunk);
        if (zb >= ze) continue;
        if (zb < sp.out_lo + r) ++n_lo;
        if (ze > sp.out_hi - r) ++n_hi;
      }
      n_lo *= tiles; n_hi *= tiles;
      unsigned long long* mine = static_cast<unsigned long long*>(p->counters.ptr);
      if (p->has_lo) {
        sp.push_lo = p->peer_ab[0][ob] + p->nzl * plane;     // my planes [G, G+r) -> its [G+nzl, ...)
        sp.band_lo = sp.out_lo + r;
        sp.sig_lo = p->peer_ctr[0] + 1;                       // "from hi" on the lo neighbour
        sp.wait_lo = mine + 0;                                // the lo neighbour pushed its hi band
        sp.wait_lo_target = (unsigned long long)(p->fused_runs * n_hi);
      }
      if (p->has_hi) {
        sp.push_hi = p->peer_ab[1][ob] - p->nzl * plane;     // my planes [G+nzl-r, G+nzl) -> its [G-r, G)
        sp.band_hi = sp.out_hi - r;
        sp.sig_hi = p->peer_ctr[1] + 0;
        sp.wait_hi = mine + 1;
        sp.wait_hi_target = (unsigned long long)(p->fused_runs * n_lo);
      }
      ++p->fused_runs;
    }
    CK(k->launch(km, sp, grid, nslot, smem, p->stream), "sweep kernel launch");
    ++launches;
    tiled_launches += tiled ? 1 : 0;
    prev = new_prev; cur = new_cur;
    j += steps;
  }
  if (p->timing) {
    CK(cudaEventRecord(t_ev1, p->stream), "timing event");
    ++p->ev_used;
    p->last_launches += launches;
    p->last_tiled += tiled_launches;
  }

  // honour the contract: (u_prev, u_cur) buffers hold (u^{n+nt-1}, u^{n+nt})
  const size_t field_bytes = (size_t)plane * p->Z * 4;
  p->last_swapped = false;
  if (prev == 0 && cur == 1) {
    // done
  } else if (prev == 1 && cur == 0 && ((c.flags & ST_NO_SWAP) || internal)) {
    p->last_swapped = true;            // the caller exchanges its references (stencil_swapped)
  } else if (prev == 1 && cur == 0) {
    const long long n4 = (long long)(field_bytes / 16);
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)p->sm_count * 8);
    swap_kernel<<<blocks, 256, 0, p->stream>>>(reinterpret_cast<float4*>(u_prev), reinterpret_cast<float4*>(u_cur), n4);
    CK(cudaGetLastError(), "swap kernel launch");
    ++aux_launches;
  } else {
    CK(cudaMemcpyAsync(u_prev, bufs[prev], field_bytes, cudaMemcpyDeviceToDevice, p->stream), "copy u_prev");
    CK(cudaMemcpyAsync(u_cur, bufs[cur], field_bytes, cudaMemcpyDeviceToDevice, p->stream), "copy u_cur");
  }
  if (p->timing) p->last_aux += aux_launches;
  return ST_OK;
}

// ------------------------------------------------------------------ library-owned exchange (a9)
// NCCL point-to-point of contiguous ghost-plane slabs (z is the slowest axis): my first / last
// `d_cur` planes of `cur` (and `d_prev` of `prev`) go to the lo / hi neighbour's ghost zone, theirs
// into mine.  Ordered after the work queued on the plan stream, and the plan stream waits for it.
static st_status nccl_chk(stencil_plan* p, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return ST_OK;
  p->broken = true;
  return fail(p, ST_ENCCL, "%s: %s", what, nccl().errstr(r));
}

static st_status exchange_slabs(stencil_plan* p, float* prev, float* cur, long long d_cur, long long d_prev,
                                bool join) {
  const NcclApi& api = nccl();
  const long long plane = p->X * p->Y;
  const long long G = p->G, nzl = p->nzl;
  const int lo = p->cfg.rank - 1, hi = p->cfg.rank + 1;
  CK(cudaEventRecord(p->ev_ready, p->stream), "exchange event");
  CK(cudaStreamWaitEvent(p->comm_stream, p->ev_ready, 0), "exchange wait");
  st_status s = nccl_chk(p, api.gstart(), "ncclGroupStart");
  if (s != ST_OK) return s;
  float* fld[2] = {cur, prev};
  const long long dep[2] = {d_cur, d_prev};
  for (int f = 0; f < 2; ++f) {
    const long long d = dep[f];
    if (d <= 0) continue;
    const size_t cnt = (size_t)(d * plane);
    if (p->has_lo) {
      if ((s = nccl_chk(p, api.send(fld[f] + G * plane, cnt, ncclFloat, lo, p->comm, p->comm_stream), "ncclSend")) != ST_OK) return s;
      if ((s = nccl_chk(p, api.recv(fld[f] + (G - d) * plane, cnt, ncclFloat, lo, p->comm, p->comm_stream), "ncclRecv")) != ST_OK) return s;
    }
    if (p->has_hi) {
      if ((s = nccl_chk(p, api.send(fld[f] + (G + nzl - d) * plane, cnt, ncclFloat, hi, p->comm, p->comm_stream), "ncclSend")) != ST_OK) return s;
      if ((s = nccl_chk(p, api.recv(fld[f] + (G + nzl) * plane, cnt, ncclFloat, hi, p->comm, p->comm_stream), "ncclRecv")) != ST_OK) return s;
    }
  }
  if ((s = nccl_chk(p, api.gend(), "ncclGroupEnd")) != ST_OK) return s;
  CK(cudaEventRecord(p->ev_done, p->comm_stream), "exchange event");
  if (join) CK(cudaStreamWaitEvent(p->stream, p->ev_done, 0), "exchange join");
  return ST_OK;
}

// stencil_run with the library-owned exchange: T_c-step periods; at T_c = T_k = 1 each step sweeps
// its boundary bands first, sends them on the comm stream while the interior is swept, and the
// next step waits for the transfer.
static st_status run_lib(stencil_plan* p, float* u_prev, float* u_cur, const float* vel,
                         const float* damp, int32_t nt, int64_t step0, int32_t nsrc,
                         const int32_t* src_xyz, const float* src_wavelet, int32_t nrec,
                         const int32_t* rec_xyz, float* rec_trace) {
  if (p->broken) return fail(p, ST_ESTATE, "plan is in an error state after an earlier fault");
  if (!u_prev || !u_cur || u_prev == u_cur) return fail(p, ST_EINVAL, "u_prev/u_cur NULL or aliased");
  if (nt < 0) return fail(p, ST_EINVAL, "nt < 0");
  if (nrec > 0 && !rec_trace) return fail(p, ST_EINVAL, "receivers need rec_trace");
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  const st_config& c = p->cfg;
  const int r = c.radius;
  if (nrec > 0) CK(cudaMemsetAsync(rec_trace, 0, (size_t)nt * nrec * 4, p->stream), "trace reset");
  float* A = u_prev;   // u^{n-1}
  float* B = u_cur;    // u^n
  const bool overlap = c.t_comm <= 1 && c.t_kernel == 1 && p->nzl >= 2 * r;
  const int G = (int)p->G, nzl = (int)p->nzl;
  bool first = true;
  st_status s = ST_OK;
  const int tc = std::max(1, c.t_comm);
  for (int done = 0; done < nt;) {
    const int steps = std::min(tc, nt - done);
    const float* v = first ? vel : nullptr;
    const float* d = first ? damp : nullptr;
    float* tr = nrec > 0 ? rec_trace + (size_t)done * nrec : nullptr;
    if (first || !overlap) {   // ghost planes of the state this period starts from
      s = exchange_slabs(p, A, B, (long long)r * steps, (long long)r * (steps - 1), true);
      if (s != ST_OK) return s;
    }
    if (overlap) {
      // bands [G, G+r) and [G+nzl-r, G+nzl) first (their new level goes to the neighbours), then
      // the interior concurrently with the transfer; T = 1 writes u^{n+1} over u^{n-1} (buffer A)
      const int ilo = p->has_lo ? G + r : G, ihi = p->has_hi ? G + nzl - r : G + nzl;
      const float* vv = v;     // the medium is derived by the first launch of the run only
      const float* dd = d;
      auto sweep = [&](int zlo, int zhi) {
        const st_status t = run_impl(p, A, B, vv, dd, 1, step0 + done, nsrc, src_xyz, src_wavelet, nrec,
                                     rec_xyz, tr, 0, nullptr, 0, zlo, zhi, true);
        vv = dd = nullptr;
        return t;
      };
      if (p->has_lo && (s = sweep(G, G + r)) != ST_OK) return s;
      if (p->has_hi && (s = sweep(G + nzl - r, G + nzl)) != ST_OK) return s;
      if ((s = exchange_slabs(p, B, A, r, 0, false)) != ST_OK) return s;   // new level A: depth r
      if (ilo < ihi && (s = sweep(ilo, ihi)) != ST_OK) return s;
      CK(cudaStreamWaitEvent(p->stream, p->ev_done, 0), "exchange join");
      std::swap(A, B);         // (u^n, u^{n+1})
    } else {
      if ((s = run_impl(p, A, B, v, d, steps, step0 + done, nsrc, src_xyz, src_wavelet, nrec, rec_xyz, tr,
                        0, nullptr, 0, -1, -1, true)) != ST_OK) return s;
      if (p->last_swapped) std::swap(A, B);
    }
    done += steps;
    first = false;
  }
  // the contract: (u_prev, u_cur) hold (u^{n+nt-1}, u^{n+nt}) -- or report the swap
  p->last_swapped = false;
  if (A != u_prev) {
    if (c.flags & ST_NO_SWAP) {
      p->last_swapped = true;
    } else {
      const long long n4 = (long long)((size_t)p->X * p->Y * p->Z * 4 / 16);
      const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)p->sm_count * 8);
      swap_kernel<<<blocks, 256, 0, p->stream>>>(reinterpret_cast<float4*>(u_prev), reinterpret_cast<float4*>(u_cur), n4);
      CK(cudaGetLastError(), "swap kernel launch");
    }
  }
  if (nrec > 0) {   // owner-only rows -> every rank gets the full trace
    CK(cudaEventRecord(p->ev_ready, p->stream), "trace event");
    CK(cudaStreamWaitEvent(p->comm_stream, p->ev_ready, 0), "trace wait");
    if ((s = nccl_chk(p, nccl().allreduce(rec_trace, rec_trace, (size_t)nt * nrec, ncclFloat, ncclSum, p->comm,
                                          p->comm_stream), "ncclAllReduce")) != ST_OK) return s;
    CK(cudaEventRecord(p->ev_done, p->comm_stream), "trace event");
    CK(cudaStreamWaitEvent(p->stream, p->ev_done, 0), "trace join");
  }
  return ST_OK;
}

st_status stencil_run(stencil_plan* p, float* u_prev, float* u_cur, const float* vel,
                      const float* damp, int32_t nt, int64_t step0, int32_t nsrc,
                      const int32_t* src_xyz, const float* src_wavelet, int32_t nrec,
                      const int32_t* rec_xyz, float* rec_trace) {
  if (p && p->comm)
    return run_lib(p, u_prev, u_cur, vel, damp, nt, step0, nsrc, src_xyz, src_wavelet, nrec, rec_xyz,
                   rec_trace);
  if (p && p->cfg.nranks == 1 && getenv("ST_SPLIT_T1") && p->cfg.t_kernel == 1 && p->nzl >= 2 * p->cfg.radius &&
      p->cfg.ndim == 3 && nt > 0) {
    // test path: every step as lo band + hi band + interior launches, the split the overlapped
    // exchange uses (no communication on one rank), so that split is checked bit for bit
    float* A = u_prev;
    float* B = u_cur;
    const int r = p->cfg.radius, G = (int)p->G, nzl = (int)p->nzl;
    for (int n = 0; n < nt; ++n) {
      float* tr = nrec > 0 ? rec_trace + (size_t)n * nrec : nullptr;
      const float* v = n == 0 ? vel : nullptr;
      const float* d = n == 0 ? damp : nullptr;
      const int cuts[4] = {G, G + r, G + nzl - r, G + nzl};
      for (int q = 0; q < 3; ++q) {
        const int lo = q == 0 ? cuts[0] : q == 1 ? cuts[2] : cuts[1];
        const int hi = q == 0 ? cuts[1] : q == 1 ? cuts[3] : cuts[2];
        if (lo >= hi) continue;
        st_status s = run_impl(p, A, B, q == 0 ? v : nullptr, q == 0 ? d : nullptr, 1, step0 + n, nsrc,
                               src_xyz, src_wavelet, nrec, rec_xyz, tr, 0, nullptr, 0, lo, hi, true);
        if (s != ST_OK) return s;
      }
      std::swap(A, B);
    }
    p->last_swapped = false;
    if (A != u_prev) {
      const long long n4 = (long long)((size_t)p->X * p->Y * p->Z * 4 / 16);
      const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)p->sm_count * 8);
      swap_kernel<<<blocks, 256, 0, p->stream>>>(reinterpret_cast<float4*>(u_prev), reinterpret_cast<float4*>(u_cur), n4);
      CK(cudaGetLastError(), "swap kernel launch");
    }
    return ST_OK;
  }
  return run_impl(p, u_prev, u_cur, vel, damp, nt, step0, nsrc, src_xyz, src_wavelet, nrec, rec_xyz,
                  rec_trace, 0, nullptr, 0);
}

static bool overlaps(const void* a, const void* b, size_t bytes) {
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return x < y + bytes && y < x + bytes;
}

st_status stencil_run_from(stencil_plan* p, const float* init_prev, const float* init_cur,
                           float* u_prev, float* u_cur, const float* vel, const float* damp,
                           int32_t nt, int64_t step0, int32_t nsrc, const int32_t* src_xyz,
                           const float* src_wavelet, int32_t nrec, const int32_t* rec_xyz,
                           float* rec_trace) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  const bool wave = p->cfg.time_order == 2;
  if (!init_cur || (wave && !init_prev)) return fail(p, ST_EINVAL, "initial field pointer is NULL");
  if (!u_prev || !u_cur) return fail(p, ST_EINVAL, "u_prev/u_cur is NULL");
  const size_t fb = (size_t)p->X * p->Y * p->Z * sizeof(float);
  // each initial field is either its own output buffer (no copy) or disjoint from both outputs
  const float* ins[2] = {wave ? init_prev : nullptr, init_cur};
  float* outs[2] = {u_prev, u_cur};
  for (int i = 0; i < 2; ++i)
    if (ins[i] && ins[i] != outs[i] && (overlaps(ins[i], u_prev, fb) || overlaps(ins[i], u_cur, fb)))
      return fail(p, ST_EINVAL, "initial field %d overlaps an output field", i);
  if (!p->comm && nt > 0 && !fused_ready(p) && res_fits(p))
    // G4: the resident kernel loads the initial pair itself (no copy, one launch)
    return run_impl(p, u_prev, u_cur, vel, damp, nt, step0, nsrc, src_xyz, src_wavelet, nrec, rec_xyz,
                    rec_trace, 0, nullptr, 0, -1, -1, false, wave ? init_prev : u_prev, init_cur);
  CK(cudaSetDevice(p->device), "cudaSetDevice");
  for (int i = 0; i < 2; ++i)
    if (ins[i] && ins[i] != outs[i])
      CK(cudaMemcpyAsync(outs[i], ins[i], fb, cudaMemcpyDeviceToDevice, p->stream), "initial field copy");
  return stencil_run(p, u_prev, u_cur, vel, damp, nt, step0, nsrc, src_xyz, src_wavelet, nrec, rec_xyz,
                     rec_trace);
}

st_status stencil_run_save(stencil_plan* p, float* u_prev, float* u_cur, const float* vel,
                           const float* damp, int32_t nt, int64_t step0, int32_t nsrc,
                           const int32_t* src_xyz, const float* src_wavelet, int32_t nrec,
                           const int32_t* rec_xyz, float* rec_trace, int32_t save_every,
                           float* snapshots, int64_t snap_stride) {
  if (!p) return fail(nullptr, ST_EINVAL, "plan is NULL");
  if (p->comm) return fail(p, ST_EUNSUPPORTED, "snapshots are not built with the library-owned exchange");
  if (save_every < 1) return fail(p, ST_EINVAL, "save_every must be >= 1 (got %d)", save_every);
  if (!snapshots && nt >= save_every) return fail(p, ST_EINVAL, "snapshots is NULL");
  if (snap_stride < p->X * p->Y * p->Z)
    return fail(p, ST_EINVAL, "snap_stride (%lld) smaller than one field (%lld floats)",
                (long long)snap_stride, (long long)(p->X * p->Y * p->Z));
  return run_impl(p, u_prev, u_cur, vel, damp, nt, step0, nsrc, src_xyz, src_wavelet, nrec, rec_xyz,
                  rec_trace, save_every, snapshots, snap_stride);
}

}  // extern "C"
