/*
 * stencil.h -- C ABI of libstencil.so, the B200 (sm_100a) time-tiled FD stencil sweep.
 *
 * What the library computes (PAPER.md = arXiv 1707.02347; "P:n" = line n of PAPER.md;
 * SURVEY.md §8 is the scope table):
 *
 *   The time-stepped explicit finite-difference star-stencil sweep Devito generates
 *   (P:519-556 diffusion, P:1671-1719 damped acoustic wave), restructured by time
 *   tiling: several time levels are computed per pass of a
 *   z-streamed on-chip window, with the streamed axis skewed by the stencil radius per
 *   level ("skew each loop ... by the negated value of the greatest
 *   negative dependence") and x-y tiles overlapped by the radius per level.
 *
 *   Per interior point p and step n (canonical order, normative):
 *       acc = K0 * u^n[p]
 *       for k = 1..r:  for axis in (x, y, z):
 *           acc = fma(W_axis_k, u^n[p - k e_axis] + u^n[p + k e_axis], acc)
 *       for each source s located at p, in index order:  acc = acc + wavelet[step0+n][s]
 *       heat (time_order 1):  u^{n+1}[p] = fma(dt, acc, u^n[p])
 *       wave (time_order 2):  u^{n+1}[p] = fma(c[p], acc, fma(a[p], u^{n-1}[p] - u^n[p], u^n[p]))
 *   with W_axis_k = (float)(coeffs[k] / dx[axis]^2), K0 = (float)(sum_axes coeffs[0]/dx[axis]^2)
 *   (double arithmetic, axes summed x, y, z), and per-point medium
 *       m = 1/(v*v),  te = (float)dt * damp,  a = (te - 2m)/(te + 2m),  c = (float)(2 dt^2)/(te + 2m)
 *   which is the paper's  u^{n+1} = ((te-2m) u^{n-1} + 4m u^n + 2dt^2 L u^n)/(te+2m)  rewritten
 *   exactly (4m/(te+2m) = 1-a).  All fp32 with denormals flushed (P:570-576 DLE flush).
 *   Points outside the global interior are zero (Dirichlet, never stored or read).
 *
 * Layout (stencil_layout): every field is fp32 [Z][Y][X], x fastest, caller-allocated:
 *     X = round_up(nx, 32)        (128-byte rows; columns >= nx are padding, never read as data)
 *     Y = ny                      (no y halo: the boundary is implicit)
 *     Z = nz_local + 2*G          (G = radius*t_comm ghost planes on each side when nranks > 1,
 *                                  G = 0 when nranks == 1; 2-D problems: Z = 1)
 *   interior point (x, y, z_local) lives at [G + z_local][y][x].
 *
 * Ownership: the caller owns every field, wavelet and trace.  The library owns the plan and
 * its device scratch (medium a/c in an interleaved layout -- 8 B per point -- plus, for the 3-D
 * wave at radius >= 3, a planar copy of a and c -- another 8 B per point -- and one flag byte
 * per tile and plane; the ping-pong pair for t_kernel > 1; source/receiver tables).  It never
 * frees caller memory.
 *
 * Errors: every entry returns st_status; nothing aborts, exits or throws across the ABI.
 * The message of the last failure is available from stencil_last_error().
 * A plan is not thread-safe: use one plan per (thread, device, stream).
 */
#ifndef PAPER_1707_02347_B200_STENCIL_H
#define PAPER_1707_02347_B200_STENCIL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stencil_plan stencil_plan;   /* opaque, owned by the library */

typedef enum {
  ST_OK = 0,
  ST_EINVAL = 1,          /* bad argument (null pointer, radius, sizes, coordinates, nt) */
  ST_ENOMEM = 2,          /* device or host allocation failed */
  ST_ECUDA = 3,           /* a CUDA runtime/driver call failed (message has the CUDA error) */
  ST_ENCCL = 4,           /* NCCL could not be loaded or a NCCL call failed (message has details) */
  ST_EUNSUPPORTED = 5,    /* (radius, t_kernel, ndim, time_order) not compiled into this build */
  ST_ESTATE = 6           /* plan is in an error state after an asynchronous failure */
} st_status;

enum {
  ST_FTZ = 1u,            /* flush denormals (required; the only arithmetic mode built) */
  ST_NO_SWAP = 2u         /* stencil_run may return the pair swapped instead of launching a swap
                             kernel (2 reads + 2 writes per point) after an odd number of in-place
                             T = 1 passes; stencil_swapped() tells the caller (see there) */
};

typedef struct {
  int32_t ndim;           /* 2 or 3 */
  int64_t n[3];           /* GLOBAL interior points (nx, ny, nz); nz = 1 when ndim == 2 */
  int32_t radius;         /* 1..8  (space order 2..16) */
  const double *coeffs;   /* host, radius+1 unscaled 2nd-derivative weights c0..cr (copied) */
  int32_t time_order;     /* 1: heat u' = u + dt*L u ; 2: damped leapfrog wave */
  double dt;
  double dx[3];           /* grid spacing per axis (dx[2] ignored for 2-D) */
  int32_t t_kernel;       /* on-chip time-tile depth T_k (1 = untiled) */
  int32_t t_comm;         /* halo depth in steps T_c (>= 1), multiple of T_k; used when nranks > 1 */
  int32_t rank, nranks;   /* z-slab index/count; n[2] % nranks == 0 */
  int32_t device;         /* CUDA device ordinal */
  void *stream;           /* cudaStream_t all work is enqueued on (NULL = legacy default) */
  uint32_t flags;         /* ST_FTZ (must be set) | ST_NO_SWAP (optional) */
  const void *nccl_id;    /* host ncclUniqueId (ST_NCCL_ID_BYTES bytes, e.g. from
                             stencil_nccl_unique_id on rank 0, broadcast by the caller) or NULL.
                             With nccl_id != NULL the LIBRARY owns the halo
                             exchange: stencil_create joins a NCCL communicator (collective: every
                             rank creates its plan concurrently), stencil_run takes any nt, loops
                             over T_c-step periods internally and sums the receiver trace over the
                             ranks (every rank gets the full trace); a one-rank plan runs the same
                             loop with no neighbours.  NULL: the caller exchanges ghost planes
                             between runs of at most t_comm steps. */
} st_config;

#define ST_NCCL_ID_BYTES 128

/* Validate cfg, pick the compiled kernel instance, allocate scratch.  *out = NULL on error.
 * Errors: ST_EINVAL (null cfg/out/coeffs, ndim, radius outside 1..8, t_kernel < 1,
 * t_comm % t_kernel != 0 when nranks > 1, n[2] % nranks != 0, rank outside [0,nranks)),
 * ST_EUNSUPPORTED (instance not built, ST_FTZ cleared), ST_ECUDA, ST_ENOMEM. */
st_status stencil_create(const st_config *cfg, stencil_plan **out);

/* padded = {X, Y, Z}; interior_origin = {0, 0, G}; z_global_range = global interior planes
 * [z0, z1) owned by this rank.  Any output pointer may be NULL. */
st_status stencil_layout(const stencil_plan *p, int64_t padded[3], int64_t interior_origin[3],
                         int64_t z_global_range[2]);

/* Advance (u_prev, u_cur) = (u^{n-1}, u^n) -> (u^{n+nt-1}, u^{n+nt}) in place.
 *   u_prev, u_cur : device, layout above, read/write.  heat: u_prev input ignored.
 *   vel, damp     : device, layout above; wave only (damp may be NULL = 0).  Must be valid on
 *                   every interior and ghost plane read (z-slabs: ghost planes included).
 *                   The run derives the medium a, c from them (one pass over vel/damp).
 *                   vel == NULL (wave): reuse the a, c of the most recent run of this plan that
 *                   passed vel (the later T_c-step chunks of one z-slab simulation); ST_ESTATE
 *                   if there was none.
 *   nt >= 0 steps; step0 = global index of the first step (indexes the wavelet rows).
 *   src_xyz       : host int32 [nsrc][3], GLOBAL interior coordinates (x, y, z)
 *   src_wavelet   : device fp32 [step0 + nt rows at least][nsrc]
 *   rec_xyz       : host int32 [nrec][3], GLOBAL interior coordinates
 *   rec_trace     : device fp32 [nt][nrec]; row n = u^{n+1} at each receiver this rank owns;
 *                   entries of receivers owned by other ranks are not written.
 * nranks > 1 without nccl_id: the caller must have exchanged ghost planes before the call (depth
 *   radius*nt of u_cur and radius*(nt-1) of u_prev), and nt <= t_comm.
 * nranks > 1 with nccl_id (library-owned exchange): any nt; every rank calls with the same nt,
 *   step0 and lists.  Each T_c period starts with a NCCL send/recv of the ghost planes on the
 *   plan's comm stream; with t_comm == t_kernel == 1 the exchange of the next level is overlapped
 *   with the interior: the r boundary planes of each side are swept first, their NCCL transfer
 *   runs on the comm stream while the interior planes are swept, and the next step waits for it.
 *   rec_trace is zeroed and then summed over the ranks (ncclAllReduce), so every rank holds it.
 * Asynchronous on cfg.stream; arguments must stay valid until it completes.
 * Source/receiver tables are rebuilt and uploaded only when src_xyz / rec_xyz differ from the
 * previous run's lists.
 * Errors: ST_EINVAL (null required pointer, nt < 0, nt > t_comm with nranks > 1, a source or
 * receiver outside the global interior), ST_ESTATE, ST_ECUDA, ST_ENOMEM. */
st_status stencil_run(stencil_plan *p, float *u_prev, float *u_cur, const float *vel,
                      const float *damp, int32_t nt, int64_t step0, int32_t nsrc,
                      const int32_t *src_xyz, const float *src_wavelet, int32_t nrec,
                      const int32_t *rec_xyz, float *rec_trace);

/* stencil_run plus snapshots of the full time dimension (the paper's "save" runs, where every
 * time level is kept; SURVEY.md §8(f) NEXT-2 ii).  For j = 1 .. floor(nt/save_every)
 * the field u^{n + j*save_every} is stored, in the field layout above, at
 *   snapshots + (j-1)*snap_stride        (device fp32, caller-owned, snap_stride >= X*Y*Z floats).
 * The store is fused into the sweep pass that produces that level (time-tiled passes are split so
 * that none crosses a snapshot step); owned planes are written, ghost planes are not.
 * Errors: as stencil_run, plus ST_EINVAL for save_every < 1, snapshots == NULL (when at least one
 * snapshot is due) or snap_stride < X*Y*Z. */
st_status stencil_run_save(stencil_plan *p, float *u_prev, float *u_cur, const float *vel,
                           const float *damp, int32_t nt, int64_t step0, int32_t nsrc,
                           const int32_t *src_xyz, const float *src_wavelet, int32_t nrec,
                           const int32_t *rec_xyz, float *rec_trace, int32_t save_every,
                           float *snapshots, int64_t snap_stride);

/* stencil_run from an initial pair that is kept: (u_prev, u_cur) receive (u^{n+nt-1}, u^{n+nt}) of
 * the run that starts from (init_prev, init_cur) = (u^{n-1}, u^n); the initial fields are not
 * modified.  Same result as copying the two fields (X*Y*Z floats each) into u_prev / u_cur and
 * calling stencil_run -- which is what it does on the plan's stream, except for the 2-D plans the
 * whole-run resident kernel serves (SURVEY §8(a) a7 taken to the end: one launch per run), where
 * that kernel loads the initial pair directly (one launch, no copy).  Use: repeated simulations
 * (the paper's timed runs) from one stored initial condition.
 *   init_prev, init_cur : device, layout above, read-only; heat: init_prev ignored (may be NULL).
 *                         Each is either its own output buffer (init_cur == u_cur: no copy) or
 *                         disjoint from both u_prev and u_cur.
 *   the other arguments : as stencil_run.
 * Errors: as stencil_run, plus ST_EINVAL for a NULL initial field or an initial field that
 * overlaps an output field it is not identical to.  On an error reported after the copies were
 * enqueued, u_prev / u_cur hold the initial pair. */
st_status stencil_run_from(stencil_plan *p, const float *init_prev, const float *init_cur,
                           float *u_prev, float *u_cur, const float *vel, const float *damp,
                           int32_t nt, int64_t step0, int32_t nsrc, const int32_t *src_xyz,
                           const float *src_wavelet, int32_t nrec, const int32_t *rec_xyz,
                           float *rec_trace);

/* 1 if the last stencil_run / stencil_run_save of p (created with ST_NO_SWAP) left the pair
 * swapped: u_prev then holds u^{n+nt} and u_cur holds u^{n+nt-1}, and the caller exchanges its two
 * references before the next run.  0 otherwise (always 0 without ST_NO_SWAP); -1 if p is NULL.
 * Used by the z-slab runner, which advances T_c = 1 step per call (an odd pass count every call). */
int32_t stencil_swapped(const stencil_plan *p);

/* ---- Fused halo push -------------------------------
 * For z-slab plans with t_comm == t_kernel == 1 and ST_NO_SWAP, the halo exchange can be fused
 * into the sweep: each T = 1 pass stores its r lowest (highest) owned output planes, besides
 * locally, straight into the lo (hi) neighbour's ghost zone over peer memory (NVLink P2P), then
 * the CTAs that pushed bump the neighbour's inbound counter (release, system scope); before the
 * TMA loads of its ghost planes the next pass waits until its own counters show the neighbours'
 * pushes of the previous step (acquire, system scope).  No NCCL call and no copy per step.
 * The ranks must issue identical run sequences (nt == 1 each) on identically configured plans;
 * the ghost planes of the first run come from the caller (initial state or one NCCL exchange).
 * Peer device pointers come from the same process (another plan of this process) or from
 * stencil_ipc_open of a blob a peer process made with stencil_ipc_export. */

/* This plan's two inbound push counters (device u64 [2]: [0] from the lo neighbour, [1] from the
 * hi neighbour), allocated and zeroed on the first call; the neighbours register them. */
st_status stencil_peer_counters(stencil_plan *p, unsigned long long **counters);

/* Register the neighbour on `side` (0 = rank-1, 1 = rank+1): my_a/my_b are this rank's two field
 * buffers (the u_prev/u_cur pair, in either order later), peer_a/peer_b the neighbour's
 * corresponding buffers (its my_a/my_b) and peer_counters its stencil_peer_counters.  Every
 * existing side must be registered before a run is fused; each registration restarts the step
 * count and zeroes this plan's inbound counter of that side (synchronously), so register only
 * while no run is in flight on this rank or its neighbours (e.g. between a device sync and a
 * barrier of all ranks).  ST_EINVAL: not a fused-capable plan (see above), no neighbour on that
 * side, null or aliased pointers, a my_a/my_b pair differing from the other side's. */
st_status stencil_set_peer(stencil_plan *p, int32_t side, const float *my_a, const float *my_b,
                           float *peer_a, float *peer_b, unsigned long long *peer_counters);

#define ST_IPC_BYTES 72
/* Export the device allocation holding dev_ptr for another process: blob (ST_IPC_BYTES) receives
 * a cudaIpcMemHandle_t of the allocation's base and the offset of dev_ptr in it. */
st_status stencil_ipc_export(const stencil_plan *p, const void *dev_ptr, void *blob);
/* Open a blob from stencil_ipc_export in this process: *dev_ptr = base + offset.  The plan
 * closes the handle when it is destroyed. */
st_status stencil_ipc_open(stencil_plan *p, const void *blob, void **dev_ptr);

/* Wait for the plan's stream; surfaces asynchronous CUDA errors (then ST_ECUDA, and the plan
 * enters ST_ESTATE). */
st_status stencil_sync(stencil_plan *p);

/* Frees scratch; NULL-safe; never touches caller memory. */
void stencil_destroy(stencil_plan *p);

/* Last error message of p, or (p == NULL) the thread-local message of the last failed
 * stencil_create / argument check.  Never NULL. */
const char *stencil_last_error(const stencil_plan *p);

/* Kernel timing (measurement support).  enable != 0: every later stencil_run
 * records CUDA events on the plan's stream immediately before its first and after its last
 * sweep-kernel launch (no host synchronisation).  stencil_timing waits for the latest end event
 * and returns, summed over every run since the previous stencil_timing (or stencil_set_timing)
 * call, the elapsed milliseconds between each run's events, the number of sweep launches, how
 * many of those were time-tiled (t_kernel-level) passes, and how many auxiliary kernels (medium
 * precompute, final swap) the runs launched; then it resets the sums.  ST_ESTATE if timing was
 * not enabled or no run has been timed since.  Any output pointer may be NULL. */
st_status stencil_set_timing(stencil_plan *p, int32_t enable);
st_status stencil_timing(stencil_plan *p, float *sweep_ms, int32_t *sweep_launches,
                         int32_t *tiled_launches, int32_t *aux_launches);

/* Pure host query (no device needed): is (ndim, time_order, radius, t_kernel) compiled? */
int32_t stencil_supported(int32_t ndim, int32_t time_order, int32_t radius, int32_t t_kernel);

/* Pure host query: library ABI version (major*100 + minor). */
int32_t stencil_abi_version(void);

/* Fill out[ST_NCCL_ID_BYTES] with a fresh ncclUniqueId (ncclGetUniqueId of the NCCL the process
 * has loaded, dlopen'ed as libnccl.so.2 or $ST_NCCL_LIB).  Host only; ST_ENCCL if NCCL is not
 * available.  Rank 0 calls it and passes the bytes to every rank's st_config.nccl_id. */
st_status stencil_nccl_unique_id(void *out);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_1707_02347_B200_STENCIL_H */
