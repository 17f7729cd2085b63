// Per-mode tridiagonal (Thomas) solves along z — kernel (c) of the north
// star, replacing tridiag._sweep (reference tridiag.py:126-167) with the
// plane-operator eigenvalues fused in (stencil.eigenvalue_plane,
// stencil.py:226-234).
//
// One thread per sine mode (m, n); consecutive threads take consecutive n,
// so every z-level access is a coalesced row segment. Eigenvalues are
// generated on the fly from the per-level weights (4a, 2b, 2c, d) and the
// mode cosines: lambda = 4a cx cy + 2b cx + 2c cy + d. The forward sweep
// stores the super-diagonal ratios cp in a workspace of the slab's size
// (tridiag.py:153 `cp = np.empty_like(w)`); the back substitution reads them.
//
// Pivot screening (tridiag.py:142-151): |denom| < threshold latches the key
// (l, m, n) with an atomicMin, so the reported failure is the first row l,
// then the smallest m, then the smallest n — np.argwhere order.
#include "hfb_internal.cuh"

namespace hfb {

__device__ __forceinline__ double eig(const double* __restrict__ co, double cx, double cy,
                                      double cxy) {
  // co = (4a, 2b, 2c, d) of one level
  const double2 w0 = __ldg(reinterpret_cast<const double2*>(co));
  const double2 w1 = __ldg(reinterpret_cast<const double2*>(co) + 1);
  (void)cxy;
  return fma(eig_p(w0.x, w1.x, cx), cy, eig_q(w0.y, w1.y, cx));
}

__device__ __forceinline__ double rcp(double d) { return rcp_fast(d); }

__device__ __forceinline__ void latch(unsigned long long* err, long long l, long long m,
                                      long long n, long long ny_total, long long nx) {
  const unsigned long long key =
      ((unsigned long long)l * (unsigned long long)ny_total + (unsigned long long)m) *
          (unsigned long long)nx +
      (unsigned long long)n;
  atomicMin(err, key);
}

struct ThomasArgs {
  int nz, nrows, ncols, nx, ny_total, m_off, swap;
  long long ld, ps;   // row stride and plane stride of the data
  long long nmodes;   // nrows * ncols
  const double* coef;
  const double* cx;
  const double* cy;
  double thr;
  unsigned long long* err;
};

// Thread per mode. Natural layout (swap = 0): rows are y-modes m_off + r,
// columns x-modes n. Transposed layout (swap = 1, the (l, n, m) order of the
// two-pass transform): rows are x-modes n, columns y-modes m.
constexpr int KCP = 8;  // cp checkpoint interval (levels)

__global__ void __launch_bounds__(256) thomas_slab_kernel(double* __restrict__ w,
                                                           double* __restrict__ cpw,
                                                           ThomasArgs a) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= a.nmodes) return;
  const int r = (int)(t / a.ncols), col = (int)(t - (long long)r * a.ncols);
  const int n = a.swap ? r : col;
  const int m = a.swap ? col : a.m_off + r;
  const double cxv = __ldg(&a.cx[n]);
  const double cyv = __ldg(&a.cy[m]);
  const double cxy = cxv * cyv;
  const long long P = a.ps;
  const long long t0 = (long long)r * a.ld + col;
  // Forward elimination. cp depends on the matrix only, so it is stored just
  // at the last level of every block of KCP levels (cpw slot = l / KCP) and
  // recomputed, bit for bit, block by block during the back substitution.
  double den = eig(a.coef + 4, cxv, cyv, cxy);
  if (fabs(den) < a.thr) latch(a.err, 0, m, n, a.ny_total, a.nx);
  double rr = rcp(den);
  double c = eig(a.coef + 8, cxv, cyv, cxy) * rr;
  // streamed data is evict-first (__ldcs/__stcs) so the per-level weights stay
  // in L1 for every mode of the CTA
  double x = __ldcs(w + t0) * rr;
  __stcs(w + t0, x);
  if (KCP == 1 && a.nz > 1) cpw[t0] = c;
  // the right-hand sides do not depend on the recurrence: keep KCP loads in
  // flight (a register ring refilled KCP levels ahead)
  double ring[KCP];
#pragma unroll
  for (int i = 0; i < KCP; ++i)
    ring[i] = (1 + i < a.nz) ? __ldcs(w + (long long)(1 + i) * P + t0) : 0.0;
  // the eigenvalues of level l + 1 are generated while level l is eliminated
  // (they do not depend on the recurrence either)
  double lo_n = 0.0, di_n = 0.0, up_n = 0.0;
  if (a.nz > 1) {
    lo_n = eig(a.coef + 12, cxv, cyv, cxy);
    di_n = eig(a.coef + 16, cxv, cyv, cxy);
    up_n = eig(a.coef + 20, cxv, cyv, cxy);
  }
  for (int l = 1; l < a.nz; ++l) {
    const long long o = (long long)l * P + t0;
    const double wl = ring[0];
#pragma unroll
    for (int i = 0; i < KCP - 1; ++i) ring[i] = ring[i + 1];
    ring[KCP - 1] = (l + KCP < a.nz) ? __ldcs(w + (long long)(l + KCP) * P + t0) : 0.0;
    const double lo = lo_n, di = di_n, up = up_n;
    if (l + 1 < a.nz) {
      const double* cn = a.coef + (long long)(l + 1) * 12;
      lo_n = eig(cn, cxv, cyv, cxy);
      di_n = eig(cn + 4, cxv, cyv, cxy);
      up_n = eig(cn + 8, cxv, cyv, cxy);
    }
    den = fma(-lo, c, di);
    if (fabs(den) < a.thr) latch(a.err, l, m, n, a.ny_total, a.nx);
    rr = rcp(den);
    x = fma(-lo, x, wl) * rr;
    __stcs(w + o, x);
    if (l < a.nz - 1) {
      c = up * rr;
      if ((l % KCP) == KCP - 1) cpw[(long long)(l / KCP) * P + t0] = c;
    }
  }
  // back substitution over blocks [b*KCP, b*KCP + KCP), descending; x = W[nz-1]
  const int bmax = (a.nz - 2) / KCP;
  double wb[KCP], cnext = 0.0;
  if (bmax >= 0) {
#pragma unroll
    for (int i = 0; i < KCP; ++i) {
      const int l = bmax * KCP + i;
      wb[i] = (l < a.nz - 1) ? __ldcs(w + (long long)l * P + t0) : 0.0;
    }
    cnext = (bmax > 0) ? cpw[(long long)(bmax - 1) * P + t0] : 0.0;
  }
  for (int b = bmax; b >= 0; --b) {
    const int l0 = b * KCP;
    double cb[KCP], wcur[KCP];
    double cprev = cnext;
#pragma unroll
    for (int i = 0; i < KCP; ++i) wcur[i] = wb[i];
    if (b > 0) {  // prefetch the next (lower) block while this one is recomputed
#pragma unroll
      for (int i = 0; i < KCP; ++i) wb[i] = __ldcs(w + (long long)(l0 - KCP + i) * P + t0);
      cnext = (b > 1) ? cpw[(long long)(b - 2) * P + t0] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < KCP; ++i) {
      const int l = l0 + i;
      if (l < a.nz - 1) {
        const double* co = a.coef + (long long)l * 12;
        const double dl = (l == 0) ? eig(co + 4, cxv, cyv, cxy)
                                   : fma(-eig(co, cxv, cyv, cxy), cprev,
                                         eig(co + 4, cxv, cyv, cxy));
        cprev = eig(co + 8, cxv, cyv, cxy) * rcp(dl);
        cb[i] = cprev;
      }
    }
#pragma unroll
    for (int i = KCP - 1; i >= 0; --i) {
      const int l = l0 + i;
      if (l < a.nz - 1) {
        x = fma(-cb[i], x, wcur[i]);
        __stcs(w + (long long)l * P + t0, x);
      }
    }
  }
}

static int launch_thomas_layout(hfb_plan* p, double* data, double* cpw, int nrows, int ncols,
                                long long ld, long long ps, int m_off, int swap,
                                cudaStream_t st) {
  if (nrows <= 0 || ncols <= 0) return HFB_OK;
  ThomasArgs a;
  a.nz = p->nz;
  a.nrows = nrows;
  a.ncols = ncols;
  a.nx = p->nx;
  a.ny_total = p->ny;
  a.m_off = m_off;
  a.swap = swap;
  a.ld = ld;
  a.ps = ps;
  a.nmodes = (long long)nrows * ncols;
  a.coef = p->coef;
  a.cx = p->cx;
  a.cy = p->cy;
  a.thr = p->thr;
  a.err = p->err;
  const long long blocks = (a.nmodes + 255) / 256;
  thomas_slab_kernel<<<(unsigned)blocks, 256, 0, st>>>(data, cpw, a);
  HFB_LAUNCHED();
  return HFB_OK;
}

int launch_thomas(hfb_plan* p, double* slab, int mloc, int m_off, double* cpw, cudaStream_t st) {
  return launch_thomas_layout(p, slab, cpw, mloc, p->nx, p->nx, (long long)mloc * p->nx, m_off,
                              0, st);
}


}  // namespace hfb

// ----------------------------------------------------------------------
// Batched Thomas on explicit bands (tridiag.solve_system, tridiag.py:59-90).
// Arrays are (nsys, n) real or (nsys, n) complex interleaved (re, im).
// thr[s] = PIVOT_RTOL * band scale of system s; the first failing row of
// each system is latched as s * n + row (min over systems).
namespace hfb {

template <bool CPLX>
struct Num;
template <>
struct Num<false> {
  typedef double T;
  static __device__ T ld(const double* p, long long i) { return p[i]; }
  static __device__ void st(double* p, long long i, T v) { p[i] = v; }
  static __device__ T sub(T a, T b) { return a - b; }
  static __device__ T mul(T a, T b) { return a * b; }
  static __device__ T div(T a, T b) { return a / b; }
  static __device__ double mag(T a) { return fabs(a); }
};
template <>
struct Num<true> {
  typedef double2 T;
  static __device__ T ld(const double* p, long long i) {
    return reinterpret_cast<const double2*>(p)[i];
  }
  static __device__ void st(double* p, long long i, T v) { reinterpret_cast<double2*>(p)[i] = v; }
  static __device__ T sub(T a, T b) { return csub(a, b); }
  static __device__ T mul(T a, T b) { return cmul(a, b); }
  static __device__ T div(T a, T b) {
    const double s = 1.0 / fma(b.x, b.x, b.y * b.y);
    return make_double2(fma(a.x, b.x, a.y * b.y) * s, fma(a.y, b.x, -a.x * b.y) * s);
  }
  static __device__ double mag(T a) { return hypot(a.x, a.y); }
};

template <bool CPLX>
__global__ void bands_kernel(const double* __restrict__ sub, const double* __restrict__ diag,
                             const double* __restrict__ sup, double* __restrict__ x,
                             double* __restrict__ cpw, int n, int nsys,
                             const double* __restrict__ thr, unsigned long long* err) {
  typedef Num<CPLX> K;
  typedef typename K::T T;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  const long long b = (long long)s * n;
  T c = K::ld(sup, b), den = K::ld(diag, b), xv;
  bool bad = K::mag(den) < thr[s];
  long long first = bad ? 0 : -1;
  c = K::div(c, den);
  xv = K::div(K::ld(x, b), den);
  K::st(cpw, b, c);
  K::st(x, b, xv);
  for (int l = 1; l < n; ++l) {
    const T lo = K::ld(sub, b + l);
    den = K::sub(K::ld(diag, b + l), K::mul(lo, c));
    if (first < 0 && K::mag(den) < thr[s]) first = l;
    if (l < n - 1) {
      c = K::div(K::ld(sup, b + l), den);
      K::st(cpw, b + l, c);
    }
    xv = K::div(K::sub(K::ld(x, b + l), K::mul(lo, xv)), den);
    K::st(x, b + l, xv);
  }
  for (int l = n - 2; l >= 0; --l) {
    xv = K::sub(K::ld(x, b + l), K::mul(K::ld(cpw, b + l), xv));
    K::st(x, b + l, xv);
  }
  if (first >= 0) atomicMin(err, (unsigned long long)(b + first));
}

}  // namespace hfb

extern "C" int hfb_solve_bands(const double* sub, const double* diag, const double* sup,
                               double* x, double* cpw, int n, int nsys, int is_complex,
                               const double* thr, unsigned long long* err, void* stream) {
  if (!sub || !diag || !sup || !x || !cpw || !thr || !err || n < 1 || nsys < 0)
    return HFB_ERR_ARGUMENT;
  if (nsys == 0) return HFB_OK;
  const int blocks = (nsys + 127) / 128;
  if (is_complex)
    hfb::bands_kernel<true><<<blocks, 128, 0, (cudaStream_t)stream>>>(sub, diag, sup, x, cpw, n,
                                                                       nsys, thr, err);
  else
    hfb::bands_kernel<false><<<blocks, 128, 0, (cudaStream_t)stream>>>(sub, diag, sup, x, cpw, n,
                                                                        nsys, thr, err);
  HFB_LAUNCHED();
  return HFB_OK;
}
