// =============================================================================
// oracle.cpp -- CPU ORACLE for the time-stepped FD stencil sweep.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load this library.  It
// shares no code, header, table or constant generator with the CUDA product
// (paper_1707_02347_b200/); the only common input is workloads/ (seeded inputs).
//
// What it computes (citations are PAPER.md lines, "P:n"):
//
//  * oracle_medium_*   per-point medium coefficients of the damped leapfrog
//                      (rewritten exactly):
//                        m  = 1/(v*v)            (squared slowness)
//                        te = dt*eta             ("tcse0 = 3.04F*damp")
//                        a  = (te - 2m)/(te + 2m)
//                        c  = 2 dt^2 /(te + 2m)
//                      so that u^{n+1} = a(u^{n-1}-u^n) + u^n + c*L_h u^n, which is
//                      the paper's ((te-2m)u^{n-1} + 4m u^n + 2dt^2 L_h u^n)/(te+2m)
//                      because 4m/(te+2m) = 1 - a.
//
//  * O1 oracle_run_untiled_*   the plain untiled loop nest of P:1671-1719 (wave)
//                      and P:519-556 (diffusion):  for n: for z: for y: for x:
//                      update(point).  This is "the plain definition" (SURVEY
//                      §8(c) O1): time tiling must reproduce it exactly.
//
//  * O1-literal oracle_run_literal_*  the same loop nest with the paper's printed update
//                      expression and term order, fp32: bounds the drift of the
//                      canonical order against the paper's own (reading Q8); not the reference.
//
//  * O3 oracle_run_slabs_*  emulation of the GPU's z-slab schedule (ghost zones of depth r*T_c,
//                      exchange every T_c steps, shrinking redundant regions): bitwise O1.
//
//  * O2 oracle_run_skewed_*    the paper's time-tiled schedule:
//                      loop order tt, zz, yy, t, z', y', x with the tiled
//                      (slow) axes skewed by `skew`*t (P:1196-1202, P:1445
//                      "int skew = 4*time", body index un-skewed P:1775-1778),
//                      the contiguous axis kept whole, and time
//                      levels held in a modulo-B buffer.
//
// The per-point arithmetic (normative order, R8):
//      acc = K0 * C[p]
//      for k = 1..r: for axis in (x, y, z):  acc = fma(W_axis_k, C[p-k e] + C[p+k e], acc)
//      for each source s at p (index order):  acc = acc + w_s[step]
//      heat: N[p] = fma(dt, acc, C[p])
//      wave: N[p] = fma(c[p], acc, fma(a[p], P[p] - C[p], C[p]))
// with W_axis_k = (T)(coef_k / h_axis^2) and K0 = (T)(sum_axes coef_0/h_axis^2)
// evaluated in double.  Denormals are flushed (FTZ/DAZ) when `ftz` != 0,
// mirroring the paper's DLE denormal flush.
//
// Oracle array layout (its own, NOT the product's): [NZ][NY][NX] with a halo of
// r on every side, NX = nx+2r, NY = ny+2r, NZ = nz+2r (3-D) or 1 (2-D).  Halo
// cells are read (they must hold zeros, Dirichlet) and never written.
// =============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <xmmintrin.h>
#include <pmmintrin.h>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct Geo {
  int ndim, r;
  long nx, ny, nz;       // interior
  long NX, NY, NZ;       // with halo
  long sy, sz;           // strides
  long zoff;             // halo offset in z (r for 3-D, 0 for 2-D)
  Geo(int ndim_, long nx_, long ny_, long nz_, int r_) : ndim(ndim_), r(r_), nx(nx_), ny(ny_), nz(nz_) {
    NX = nx + 2 * r; NY = ny + 2 * r;
    NZ = (ndim == 3) ? nz + 2 * r : 1;
    zoff = (ndim == 3) ? r : 0;
    sy = NX; sz = NX * NY;
  }
  long idx(long x, long y, long z) const { return (z + zoff) * sz + (y + r) * sy + (x + r); }
  long total() const { return NZ * sz; }
};

template <class T>
struct Coef {
  T K0;
  T W[3][17];            // W[axis][k], k = 1..r
};

template <class T>
Coef<T> make_coef(const Geo& g, const double* coeffs, const double* h) {
  Coef<T> cf{};
  double k0 = 0.0;
  for (int a = 0; a < g.ndim; ++a) k0 += coeffs[0] / (h[a] * h[a]);
  cf.K0 = (T)k0;
  for (int a = 0; a < g.ndim; ++a)
    for (int k = 1; k <= g.r; ++k) cf.W[a][k] = (T)(coeffs[k] / (h[a] * h[a]));
  return cf;
}

struct FtzGuard {   // per-thread MXCSR FTZ|DAZ
  unsigned old;
  bool on;
  explicit FtzGuard(int ftz) : old(_mm_getcsr()), on(ftz != 0) {
    if (on) _mm_setcsr(old | 0x8040u);
  }
  ~FtzGuard() { if (on) _mm_setcsr(old); }
};

inline float fmaT(float a, float b, float c) { return std::fmaf(a, b, c); }
inline double fmaT(double a, double b, double c) { return std::fma(a, b, c); }

// Sources/receivers of one problem, as oracle-layout linear indices.
struct PointList {
  std::vector<long> p;      // linear index
  std::vector<long> z, y;   // interior z, y (for fast row filtering)
};

PointList make_points(const Geo& g, int n, const int64_t* xyz) {
  PointList L;
  for (int i = 0; i < n; ++i) {
    long x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    L.p.push_back(g.idx(x, y, z));
    L.y.push_back(y);
    L.z.push_back(z);
  }
  return L;
}

// The canonical per-point update.  `src_acc` adds the sources located at p, in index order.
template <class T>
inline T update_point(const Geo& g, const Coef<T>& cf, int time_order, T dtT,
                      const T* C, const T* Pold, const T* a, const T* c, long p,
                      const PointList& S, const T* w_step, long y, long z, bool row_has_src) {
  T acc = cf.K0 * C[p];
  for (int k = 1; k <= g.r; ++k) {
    acc = fmaT(cf.W[0][k], C[p - k] + C[p + k], acc);
    acc = fmaT(cf.W[1][k], C[p - k * g.sy] + C[p + k * g.sy], acc);
    if (g.ndim == 3) acc = fmaT(cf.W[2][k], C[p - k * g.sz] + C[p + k * g.sz], acc);
  }
  if (row_has_src) {
    for (size_t s = 0; s < S.p.size(); ++s)
      if (S.p[s] == p) acc = acc + w_step[s];
  }
  (void)y; (void)z;
  if (time_order == 1) return fmaT(dtT, acc, C[p]);
  return fmaT(c[p], acc, fmaT(a[p], Pold[p] - C[p], C[p]));
}

template <class T>
bool row_has_source(const PointList& S, long y, long z) {
  for (size_t s = 0; s < S.p.size(); ++s)
    if (S.y[s] == y && S.z[s] == z) return true;
  return false;
}

// ---------------------------------------------------------------------------- O1
template <class T>
int run_untiled(int ndim, long nx, long ny, long nz, int r, const double* coeffs, const double* h,
                int time_order, double dt, T* P, T* C, const T* a, const T* c, int nt, long step0,
                int nsrc, const int64_t* src_xyz, const T* wavelet, int nrec, const int64_t* rec_xyz,
                T* trace, int ftz) {
  if (ndim != 2 && ndim != 3) return 1;
  if (r < 1 || r > 16 || nt < 0) return 1;
  Geo g(ndim, nx, ny, nz, r);
  const Coef<T> cf = make_coef<T>(g, coeffs, h);
  const T dtT = (T)dt;
  const PointList S = make_points(g, nsrc, src_xyz);
  const PointList Rc = make_points(g, nrec, rec_xyz);
  T* bufP = P;   // u^{n-1}; receives u^{n+1}
  T* bufC = C;   // u^n
  const long nzl = (ndim == 3) ? nz : 1;
  for (int n = 0; n < nt; ++n) {
    const T* w_step = nsrc ? wavelet + (step0 + n) * nsrc : nullptr;
    T* N = bufP;
    const T* Pold = bufP;
    const T* Cc = bufC;
#pragma omp parallel
    {
      FtzGuard guard(ftz);
#pragma omp for schedule(static)
      for (long z = 0; z < nzl; ++z)
        for (long y = 0; y < ny; ++y) {
          const bool hs = nsrc && row_has_source<T>(S, y, z);
          for (long x = 0; x < nx; ++x) {
            const long p = g.idx(x, y, z);
            N[p] = update_point<T>(g, cf, time_order, dtT, Cc, Pold, a, c, p, S, w_step, y, z, hs);
          }
        }
    }
    for (int k = 0; k < nrec; ++k) trace[(long)n * nrec + k] = N[Rc.p[k]];
    std::swap(bufP, bufC);   // bufC = newest
  }
  if (nt % 2 == 1) {          // honour (u_prev, u_cur) = (u^{n+nt-1}, u^{n+nt}) in the caller's buffers
    const long tot = g.total();
    for (long i = 0; i < tot; ++i) std::swap(P[i], C[i]);
  }
  return 0;
}

// ---------------------------------------------------------------------------- O1-literal
// The paper's own expression for the damped wave update, term by term in the order printed at
// P:1678-1708 (fp32, C left-to-right evaluation, no contraction):
//     num = (tcse0 - 2m) u^{n-1}
//           + w_r S_r + w_{r-1} S_{r-1} + ... + w_1 S_1      (paper: "- 8.25e-5F*(...) + ..."),
//           + 4 m u^n  + w_0 u^n,            u^{n+1} = num / (tcse0 + 2m)
// with tcse0 = dt*damp, m = 1/v^2, w_k = (T)(2 dt^2 c_k / h^2), w_0 = (T)(2 dt^2 ndim c_0 / h^2)
// and S_k = u[c-k] + u[c+k] (contiguous axis) + u[y-k] + u[y+k] + u[slow-k] + u[slow+k], summed
// left to right (the paper's contiguous axis is its z: its "z - 4" pair comes first).
// A source term (none in the paper) enters the numerator as + (T)(2 dt^2) * w_s
// after the neighbour sums.  Isotropic spacing only (the printed form has one weight per k).
// This is a second, independently ordered evaluation used to bound the fp32 drift between the
// canonical order and the paper's order (reading Q8); it is not the parity reference.
template <class T>
int run_literal(int ndim, long nx, long ny, long nz, int r, const double* coeffs, const double* h,
                double dt, T* P, T* C, const T* vel, const T* damp, int nt, long step0,
                int nsrc, const int64_t* src_xyz, const T* wavelet, int nrec, const int64_t* rec_xyz,
                T* trace, int ftz) {
  if (ndim != 2 && ndim != 3) return 1;
  if (r < 1 || r > 16 || nt < 0) return 1;
  for (int a = 1; a < ndim; ++a) if (h[a] != h[0]) return 2;
  Geo g(ndim, nx, ny, nz, r);
  const double s2 = 2.0 * dt * dt / (h[0] * h[0]);
  T w[17];
  for (int k = 1; k <= r; ++k) w[k] = (T)(s2 * coeffs[k]);
  const T w0 = (T)(s2 * ndim * coeffs[0]);
  const T dtT = (T)dt, two_dt2 = (T)(2.0 * dt * dt);
  const PointList S = make_points(g, nsrc, src_xyz);
  const PointList Rc = make_points(g, nrec, rec_xyz);
  T* bufP = P;
  T* bufC = C;
  const long nzl = (ndim == 3) ? nz : 1;
  for (int n = 0; n < nt; ++n) {
    const T* w_step = nsrc ? wavelet + (step0 + n) * nsrc : nullptr;
    T* N = bufP;
    const T* Cc = bufC;
#pragma omp parallel
    {
      FtzGuard guard(ftz);
#pragma omp for schedule(static)
      for (long z = 0; z < nzl; ++z)
        for (long y = 0; y < ny; ++y) {
          const bool hs = nsrc && row_has_source<T>(S, y, z);
          for (long x = 0; x < nx; ++x) {
            const long p = g.idx(x, y, z);
            const T v = vel[p];
            const T m = (T)1 / (v * v);
            const T tcse0 = dtT * damp[p];
            T num = (tcse0 - (T)2 * m) * N[p];       // N[p] still holds u^{n-1}
            for (int k = r; k >= 1; --k) {
              T sk = Cc[p - k] + Cc[p + k];
              sk = sk + Cc[p - k * g.sy];
              sk = sk + Cc[p + k * g.sy];
              if (ndim == 3) { sk = sk + Cc[p - k * g.sz]; sk = sk + Cc[p + k * g.sz]; }
              num = num + w[k] * sk;
            }
            if (hs)
              for (size_t s = 0; s < S.p.size(); ++s)
                if (S.p[s] == p) num = num + two_dt2 * w_step[s];
            num = num + (T)4 * m * Cc[p];
            num = num + w0 * Cc[p];
            N[p] = num / (tcse0 + (T)2 * m);
          }
        }
    }
    for (int k = 0; k < nrec; ++k) trace[(long)n * nrec + k] = N[Rc.p[k]];
    std::swap(bufP, bufC);
  }
  if (nt % 2 == 1) {
    const long tot = g.total();
    for (long i = 0; i < tot; ++i) std::swap(P[i], C[i]);
  }
  return 0;
}

// ---------------------------------------------------------------------------- O2
// Paper's skewed, time-tiled schedule.  Tiled axes are the slow ones
// (z and y in 3-D; y in 2-D), skewed by `skew` per time step; x (contiguous) whole.
template <class T>
int run_skewed(int ndim, long nx, long ny, long nz, int r, const double* coeffs, const double* h,
               int time_order, double dt, T* P, T* C, const T* a, const T* c, int nt, long step0,
               int nsrc, const int64_t* src_xyz, const T* wavelet, int nrec, const int64_t* rec_xyz,
               T* trace, int ftz, int Tt, int Tz, int Ty, int B, int skew) {
  if (ndim != 2 && ndim != 3) return 1;
  if (Tt < 1 || Tz < 1 || Ty < 1 || B < 2 || skew < 0 || nt < 0) return 1;
  Geo g(ndim, nx, ny, nz, r);
  const Coef<T> cf = make_coef<T>(g, coeffs, h);
  const T dtT = (T)dt;
  const PointList S = make_points(g, nsrc, src_xyz);
  const PointList Rc = make_points(g, nrec, rec_xyz);
  const long tot = g.total();
  // Level L lives in buf[L % B]: level 0 = u^{n-1}, level 1 = u^n, step t writes level t+2.
  std::vector<std::vector<T>> buf(B, std::vector<T>(P, P + tot));
  std::copy(P, P + tot, buf[0].begin());
  std::copy(C, C + tot, buf[1 % B].begin());
  const long nzl = (ndim == 3) ? nz : 1;
  // recv maps: receiver k lives at oracle index Rc.p[k]
  FtzGuard guard(ftz);
  auto floordiv = [](long a_, long b_) { return (a_ >= 0) ? a_ / b_ : -((-a_ + b_ - 1) / b_); };
  for (long tt = 0; tt < nt; tt += Tt) {
    const long t_hi = std::min<long>(nt, tt + Tt);
    // skewed coordinate ranges over this time tile
    const long zs_lo = (ndim == 3) ? skew * tt : 0;
    const long zs_hi = (ndim == 3) ? (nzl - 1 + skew * (t_hi - 1)) : 0;
    const long ys_lo = skew * tt, ys_hi = ny - 1 + skew * (t_hi - 1);
    const long zz0 = (ndim == 3) ? floordiv(zs_lo, Tz) * Tz : 0;
    for (long zz = zz0; zz <= zs_hi; zz += (ndim == 3 ? Tz : 1)) {
      for (long yy = floordiv(ys_lo, Ty) * Ty; yy <= ys_hi; yy += Ty) {
        for (long t = tt; t < t_hi; ++t) {
          T* N = buf[(t + 2) % B].data();
          const T* Cc = buf[(t + 1) % B].data();
          const T* Pold = buf[t % B].data();
          const T* w_step = nsrc ? wavelet + (step0 + t) * nsrc : nullptr;
          long zlo, zhi;
          if (ndim == 3) { zlo = std::max(zz, skew * t); zhi = std::min(zz + Tz, skew * t + nzl); }
          else { zlo = 0; zhi = 1; }
          const long ylo = std::max(yy, skew * t), yhi = std::min(yy + Ty, skew * t + ny);
          for (long zsk = zlo; zsk < zhi; ++zsk) {
            const long z = (ndim == 3) ? zsk - skew * t : 0;     // un-skew
            for (long ysk = ylo; ysk < yhi; ++ysk) {
              const long y = ysk - skew * t;
              const bool hs = nsrc && row_has_source<T>(S, y, z);
              for (long x = 0; x < nx; ++x) {
                const long p = g.idx(x, y, z);
                N[p] = update_point<T>(g, cf, time_order, dtT, Cc, Pold, a, c, p, S, w_step, y, z, hs);
              }
              for (int k = 0; k < nrec; ++k)
                if (Rc.y[k] == y && Rc.z[k] == z) trace[t * nrec + k] = N[Rc.p[k]];
            }
          }
        }
      }
    }
  }
  std::copy(buf[nt % B].begin(), buf[nt % B].end(), P);
  std::copy(buf[(nt + 1) % B].begin(), buf[(nt + 1) % B].end(), C);
  return 0;
}

// ---------------------------------------------------------------------------- O3
// Emulation of the GPU's z-slab schedule, plain loops:
// the interior planes are split into S slabs; each slab keeps its own copy of the fields with
// `ghost` extra planes per side (zero at the global boundary); every T_c steps the slabs copy their
// neighbours' owned planes into their ghost zones (depth r*T_c of u^n and r*(T_c-1) of u^{n-1},
// what the library exchanges), then advance T_c steps without communication over regions that
// shrink by r per step (ghost planes are computed redundantly, sources injected there too),
// receivers sampled by the owning slab only.  Must equal O1 bit for bit whenever ghost >= r*T_c;
// a shallower ghost zone must not (negative control).
template <class T>
int run_slabs(int ndim, long nx, long ny, long nz, int r, const double* coeffs, const double* h,
              int time_order, double dt, T* P, T* C, const T* a, const T* c, int nt, long step0,
              int nsrc, const int64_t* src_xyz, const T* wavelet, int nrec, const int64_t* rec_xyz,
              T* trace, int ftz, int nslab, int tc, int ghost) {
  if (ndim != 3 || nslab < 1 || tc < 1 || ghost < 0 || nz % nslab) return 1;
  const Geo g(ndim, nx, ny, nz, r);           // the global arrays (oracle layout, halo r)
  const Coef<T> cf = make_coef<T>(g, coeffs, h);
  const T dtT = (T)dt;
  const long nzl = nz / nslab;
  const long sz = g.sz;
  FtzGuard guard(ftz);
  // slab s stores global planes [z0 - gl, z0 + nzl + gh) at local planes [0, ...), plus the
  // r-plane halo the per-point update reads beyond them (always zero)
  struct Slab { long z0, gl, gh, nloc; std::vector<T> P, C, A, Cc; };
  std::vector<Slab> sl(nslab);
  for (int s = 0; s < nslab; ++s) {
    Slab& b = sl[s];
    b.z0 = s * nzl;
    b.gl = s > 0 ? ghost : 0;
    b.gh = s < nslab - 1 ? ghost : 0;
    b.nloc = b.gl + nzl + b.gh;
    const long tot = (b.nloc + 2 * r) * sz;
    b.P.assign(tot, (T)0); b.C.assign(tot, (T)0);
    if (time_order == 2) { b.A.assign(tot, (T)0); b.Cc.assign(tot, (T)0); }
    for (long lz = 0; lz < b.nloc; ++lz) {      // state on owned planes; medium on every plane
      const long gz = b.z0 - b.gl + lz;
      for (long i = 0; i < sz; ++i) {
        const long src = (gz + r) * sz + i, dst = (lz + r) * sz + i;
        if (lz >= b.gl && lz < b.gl + nzl) { b.P[dst] = P[src]; b.C[dst] = C[src]; }
        if (time_order == 2) { b.A[dst] = a[src]; b.Cc[dst] = c[src]; }
      }
    }
  }
  // a slab-local geometry: same x/y, nloc planes
  auto local_idx = [&](long x, long y, long lz) { return (lz + r) * sz + (y + r) * g.sy + (x + r); };
  const PointList S = make_points(g, nsrc, src_xyz);
  for (long done = 0; done < nt;) {
    const long steps = std::min<long>(tc, nt - done);
    // exchange: ghost planes from the neighbours' owned planes (u^n depth r*steps, u^{n-1} r*(steps-1))
    for (int s = 0; s < nslab; ++s) {
      Slab& b = sl[s];
      const long dc = std::min<long>(r * steps, ghost), dp = std::min<long>(r * (steps - 1), ghost);
      for (int side = 0; side < 2; ++side) {
        if ((side == 0 && s == 0) || (side == 1 && s == nslab - 1)) continue;
        const Slab& nb = sl[side == 0 ? s - 1 : s + 1];
        for (int f = 0; f < 2; ++f) {
          const long d = f == 0 ? dc : dp;
          for (long k = 0; k < d; ++k) {
            // my ghost plane and the global plane it mirrors
            const long lz = side == 0 ? b.gl - 1 - k : b.gl + nzl + k;
            const long gz = b.z0 - b.gl + lz;
            const long nlz = gz - (nb.z0 - nb.gl);
            const std::vector<T>& from = f == 0 ? nb.C : nb.P;
            std::vector<T>& to = f == 0 ? b.C : b.P;
            std::copy(from.begin() + (nlz + r) * sz, from.begin() + (nlz + r + 1) * sz, to.begin() + (lz + r) * sz);
          }
        }
      }
    }
    for (long j = 0; j < steps; ++j) {
      const long n = done + j;
      const T* w_step = nsrc ? wavelet + (step0 + n) * nsrc : nullptr;
      for (int s = 0; s < nslab; ++s) {
        Slab& b = sl[s];
        const long ext = (long)r * (steps - 1 - j);
        const long lo = b.gl - (s > 0 ? std::min(ext, b.gl) : 0);
        const long hi = b.gl + nzl + (s < nslab - 1 ? std::min(ext, b.gh) : 0);
        // the per-point update reads u^n at lz +- r; a slab-local Geo view of the arrays
        Geo lg(3, nx, ny, b.nloc, r);
        for (long lz = lo; lz < hi; ++lz) {
          const long gz = b.z0 - b.gl + lz;
          for (long y = 0; y < ny; ++y) {
            const bool hs = nsrc && row_has_source<T>(S, y, gz);
            for (long x = 0; x < nx; ++x) {
              const long pl = local_idx(x, y, lz);
              // sources by global position: a one-source list per matching point
              T acc_unused = 0; (void)acc_unused;
              PointList Sl;
              if (hs)
                for (size_t q = 0; q < S.p.size(); ++q) {
                  Sl.p.push_back(S.p[q] == g.idx(x, y, gz) ? pl : -1);
                  Sl.y.push_back(S.y[q]); Sl.z.push_back(S.z[q]);
                }
              b.P[pl] = update_point<T>(lg, cf, time_order, dtT, b.C.data(), b.P.data(),
                                        time_order == 2 ? b.A.data() : nullptr,
                                        time_order == 2 ? b.Cc.data() : nullptr, pl, Sl, w_step, y, gz, hs);
            }
          }
        }
      }
      for (int k = 0; k < nrec; ++k) {           // owner-only receivers
        const long gz = rec_xyz[3 * k + 2];
        const int s = (int)(gz / nzl);
        const Slab& b = sl[s];
        trace[(long)n * nrec + k] = b.P[local_idx(rec_xyz[3 * k], rec_xyz[3 * k + 1], gz - b.z0 + b.gl)];
      }
      for (int s = 0; s < nslab; ++s) std::swap(sl[s].P, sl[s].C);
    }
    done += steps;
  }
  // gather the owned planes; (u_prev, u_cur) = (u^{n+nt-1}, u^{n+nt})
  for (int s = 0; s < nslab; ++s) {
    const Slab& b = sl[s];
    for (long lz = b.gl; lz < b.gl + nzl; ++lz) {
      const long gz = b.z0 - b.gl + lz;
      std::copy(b.P.begin() + (lz + r) * sz, b.P.begin() + (lz + r + 1) * sz, P + (gz + r) * sz);
      std::copy(b.C.begin() + (lz + r) * sz, b.C.begin() + (lz + r + 1) * sz, C + (gz + r) * sz);
    }
  }
  return 0;
}

template <class T>
void medium(long npts, const T* vel, const T* eta, double dt, T* a, T* c, int ftz) {
  const T dtT = (T)dt;
  const T two_dt2 = (T)(2.0 * dt * dt);
#pragma omp parallel
  {
    FtzGuard guard(ftz);
#pragma omp for schedule(static)
    for (long i = 0; i < npts; ++i) {
      const T v = vel[i];
      const T m = (T)1 / (v * v);
      const T te = dtT * (eta ? eta[i] : (T)0);
      const T m2 = (T)2 * m;
      const T den = te + m2;
      a[i] = (te - m2) / den;
      c[i] = two_dt2 / den;
    }
  }
}

}  // namespace

extern "C" {

int oracle_run_untiled_f32(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                           const double* h, int time_order, double dt, float* P, float* C,
                           const float* a, const float* c, int nt, long step0, int nsrc,
                           const int64_t* src_xyz, const float* wavelet, int nrec,
                           const int64_t* rec_xyz, float* trace, int ftz) {
  return run_untiled<float>(ndim, nx, ny, nz, r, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                            nsrc, src_xyz, wavelet, nrec, rec_xyz, trace, ftz);
}

int oracle_run_untiled_f64(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                           const double* h, int time_order, double dt, double* P, double* C,
                           const double* a, const double* c, int nt, long step0, int nsrc,
                           const int64_t* src_xyz, const double* wavelet, int nrec,
                           const int64_t* rec_xyz, double* trace, int ftz) {
  return run_untiled<double>(ndim, nx, ny, nz, r, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                             nsrc, src_xyz, wavelet, nrec, rec_xyz, trace, ftz);
}

int oracle_run_literal_f32(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                           const double* h, double dt, float* P, float* C, const float* vel,
                           const float* damp, int nt, long step0, int nsrc, const int64_t* src_xyz,
                           const float* wavelet, int nrec, const int64_t* rec_xyz, float* trace,
                           int ftz) {
  return run_literal<float>(ndim, nx, ny, nz, r, coeffs, h, dt, P, C, vel, damp, nt, step0, nsrc,
                            src_xyz, wavelet, nrec, rec_xyz, trace, ftz);
}

int oracle_run_literal_f64(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                           const double* h, double dt, double* P, double* C, const double* vel,
                           const double* damp, int nt, long step0, int nsrc, const int64_t* src_xyz,
                           const double* wavelet, int nrec, const int64_t* rec_xyz, double* trace,
                           int ftz) {
  return run_literal<double>(ndim, nx, ny, nz, r, coeffs, h, dt, P, C, vel, damp, nt, step0, nsrc,
                             src_xyz, wavelet, nrec, rec_xyz, trace, ftz);
}

int oracle_run_slabs_f32(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                         const double* h, int time_order, double dt, float* P, float* C,
                         const float* a, const float* c, int nt, long step0, int nsrc,
                         const int64_t* src_xyz, const float* wavelet, int nrec,
                         const int64_t* rec_xyz, float* trace, int ftz, int nslab, int tc, int ghost) {
  return run_slabs<float>(ndim, nx, ny, nz, r, coeffs, h, time_order, dt, P, C, a, c, nt, step0, nsrc,
                          src_xyz, wavelet, nrec, rec_xyz, trace, ftz, nslab, tc, ghost);
}

int oracle_run_skewed_f32(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                          const double* h, int time_order, double dt, float* P, float* C,
                          const float* a, const float* c, int nt, long step0, int nsrc,
                          const int64_t* src_xyz, const float* wavelet, int nrec,
                          const int64_t* rec_xyz, float* trace, int ftz, int Tt, int Tz, int Ty,
                          int B, int skew) {
  return run_skewed<float>(ndim, nx, ny, nz, r, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                           nsrc, src_xyz, wavelet, nrec, rec_xyz, trace, ftz, Tt, Tz, Ty, B, skew);
}

int oracle_run_skewed_f64(int ndim, long nx, long ny, long nz, int r, const double* coeffs,
                          const double* h, int time_order, double dt, double* P, double* C,
                          const double* a, const double* c, int nt, long step0, int nsrc,
                          const int64_t* src_xyz, const double* wavelet, int nrec,
                          const int64_t* rec_xyz, double* trace, int ftz, int Tt, int Tz, int Ty,
                          int B, int skew) {
  return run_skewed<double>(ndim, nx, ny, nz, r, coeffs, h, time_order, dt, P, C, a, c, nt, step0,
                            nsrc, src_xyz, wavelet, nrec, rec_xyz, trace, ftz, Tt, Tz, Ty, B, skew);
}

void oracle_medium_f32(long npts, const float* vel, const float* eta, double dt, float* a, float* c,
                       int ftz) {
  medium<float>(npts, vel, eta, dt, a, c, ftz);
}

void oracle_medium_f64(long npts, const double* vel, const double* eta, double dt, double* a,
                       double* c, int ftz) {
  medium<double>(npts, vel, eta, dt, a, c, ftz);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
