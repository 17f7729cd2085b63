// Compact-scheme RHS operators (kernel (a) of the north star), the 27-point
// operator used for the Dirichlet fold and residuals, and the z-slab <->
// y-block pack/unpack of the partitioned exchange.
//
// RHS and 27-point kernels use explicit round-to-nearest intrinsics (no FMA
// contraction) and the reference's exact term order, so for real data they
// reproduce the reference's numpy results bit for bit (the complex
// arithmetic of the reference reduces to these real operations when the
// imaginary parts are zero).
#include "hfb_internal.cuh"
#include "tma.cuh"

namespace hfb {

#define DADD __dadd_rn
#define DMUL __dmul_rn

// assembly.py:183-193: F = hz2 * (0.5*core + (xm + xp + ym + yp + zm + zp) * (1/12))
__global__ void rhs_fourth_kernel(const double* __restrict__ f, double* __restrict__ F, int nx,
                                  int ny, int nz, double hz2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y, l = blockIdx.z;
  if (i >= nx) return;
  const long long X = nx + 2, XY = (long long)(nx + 2) * (ny + 2);
  const long long c = (long long)(l + 1) * XY + (long long)(j + 1) * X + (i + 1);
  double nb = DADD(__ldg(&f[c - 1]), __ldg(&f[c + 1]));
  nb = DADD(nb, __ldg(&f[c - X]));
  nb = DADD(nb, __ldg(&f[c + X]));
  nb = DADD(nb, __ldg(&f[c - XY]));
  nb = DADD(nb, __ldg(&f[c + XY]));
  // the reference divides a complex128 array by 12.0, which numpy evaluates
  // as a product with the reciprocal 1/12
  const double v = DADD(DMUL(0.5, __ldg(&f[c])), DMUL(nb, 1.0 / 12.0));
  F[((long long)l * ny + j) * nx + i] = DMUL(hz2, v);
}

// The same operator marching up the levels: a thread owns column (i, j) for lz
// levels and slides (below, centre, above) through registers, loading the
// column one level ahead, so each level costs one new centre-column load plus
// the four in-plane neighbours; a CTA covers TX x TY columns, so the
// y-neighbour rows are its own (L1). Same term order as rhs_fourth_kernel.
template <int TX, int TY>
__global__ void __launch_bounds__(TX * TY) rhs_fourth_march_kernel(const double* __restrict__ f,
                                                                    double* __restrict__ F,
                                                                    int nx, int ny, int nz,
                                                                    double hz2, int lz) {
  const int i = blockIdx.x * TX + threadIdx.x % TX, j = blockIdx.y * TY + threadIdx.x / TX;
  if (i >= nx || j >= ny) return;
  const int l0 = blockIdx.z * lz, l1 = min(nz, l0 + lz);
  const long long X = nx + 2, XY = X * (ny + 2);
  long long c = (long long)(l0 + 1) * XY + (long long)(j + 1) * X + (i + 1);
  double zm = __ldg(&f[c - XY]), zc = __ldg(&f[c]), zn = __ldg(&f[c + XY]);
#pragma unroll 2
  for (int l = l0; l < l1; ++l, c += XY) {
    const double zp = zn;
    if (l + 1 < l1) zn = __ldg(&f[c + 2 * XY]);  // the column one level ahead
    double nb = DADD(__ldg(&f[c - 1]), __ldg(&f[c + 1]));
    nb = DADD(nb, __ldg(&f[c - X]));
    nb = DADD(nb, __ldg(&f[c + X]));
    nb = DADD(nb, zm);
    nb = DADD(nb, zp);
    const double v = DADD(DMUL(0.5, zc), DMUL(nb, 1.0 / 12.0));
    F[((long long)l * ny + j) * nx + i] = DMUL(hz2, v);
    zm = zc;
    zc = zp;
  }
}

// assembly.py:180-181
__global__ void rhs_second_kernel(const double* __restrict__ f, double* __restrict__ F,
                                  long long n, double hz2) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    F[e] = DMUL(hz2, f[e]);
}

// assembly.py:195-213 (uniform grid, h = h_z):
// rhs = h2*(f + (h2/12) lap + (h4/360) d4 + (h4/90) mixed)
//       - ((h4/20) k2) f + ((h2 h4/60) k2z) fz
__global__ void rhs_sixth_kernel(const double* __restrict__ f, const double* __restrict__ lap,
                                 const double* __restrict__ d4, const double* __restrict__ fxxyy,
                                 const double* __restrict__ fxxzz,
                                 const double* __restrict__ fyyzz,
                                 const double* __restrict__ fz, const double* __restrict__ k2,
                                 const double* __restrict__ k2z, double h2, long long plane,
                                 long long n, double* __restrict__ F) {
  const double h4 = DMUL(h2, h2);
  const double c1 = __ddiv_rn(h2, 12.0), c2 = __ddiv_rn(h4, 360.0), c3 = __ddiv_rn(h4, 90.0);
  const double c4 = __ddiv_rn(h4, 20.0), c5 = __ddiv_rn(DMUL(h2, h4), 60.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long l = e / plane;
    const double mixed = DADD(DADD(fxxyy[e], fxxzz[e]), fyyzz[e]);
    double in = DADD(f[e], DMUL(c1, lap[e]));
    in = DADD(in, DMUL(c2, d4[e]));
    in = DADD(in, DMUL(c3, mixed));
    double r = DMUL(h2, in);
    r = __dsub_rn(r, DMUL(DMUL(c4, k2[l]), f[e]));
    r = DADD(r, DMUL(DMUL(c5, k2z[l]), fz[e]));
    F[e] = r;
  }
}

// assembly.py:215-224:
// rhs = hz2*(f + (hx2/12) fxx + (hy2/12) fyy + (hz2/12)(gamma fz + fzz))
__global__ void rhs_convdiff_kernel(const double* __restrict__ f, const double* __restrict__ fxx,
                                    const double* __restrict__ fyy, const double* __restrict__ fz,
                                    const double* __restrict__ fzz, double hx2, double hy2,
                                    double hz2, double gamma, long long n,
                                    double* __restrict__ F) {
  const double a = __ddiv_rn(hx2, 12.0), b = __ddiv_rn(hy2, 12.0), c = __ddiv_rn(hz2, 12.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    double in = DADD(f[e], DMUL(a, fxx[e]));
    in = DADD(in, DMUL(b, fyy[e]));
    in = DADD(in, DMUL(c, DADD(DMUL(gamma, fz[e]), fzz[e])));
    F[e] = DMUL(hz2, in);
  }
}

// Complex variants (complex k(z) / complex gamma, complex sources): the same
// formulas in complex arithmetic with the reference's operation order —
// real coefficients scale both parts, complex products are
// (ar br - ai bi, ar bi + ai br).
struct Fields7 {
  const double* p[7];
};

__global__ void rhs_sixth_z_kernel(Fields7 fr, Fields7 fi, const double* __restrict__ k2r,
                                   const double* __restrict__ k2i,
                                   const double* __restrict__ k2zr,
                                   const double* __restrict__ k2zi, double h2, long long plane,
                                   long long n, double* __restrict__ Fr,
                                   double* __restrict__ Fi) {
  const double h4 = DMUL(h2, h2);
  const double c1 = __ddiv_rn(h2, 12.0), c2 = __ddiv_rn(h4, 360.0), c3 = __ddiv_rn(h4, 90.0);
  const double c4 = __ddiv_rn(h4, 20.0), c5 = __ddiv_rn(DMUL(h2, h4), 60.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long l = e / plane;
    double out[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const Fields7& F = c ? fi : fr;  // f, lap, d4, fxxyy, fxxzz, fyyzz, fz
      const double mixed = DADD(DADD(F.p[3][e], F.p[4][e]), F.p[5][e]);
      double in = DADD(F.p[0][e], DMUL(c1, F.p[1][e]));
      in = DADD(in, DMUL(c2, F.p[2][e]));
      in = DADD(in, DMUL(c3, mixed));
      out[c] = DMUL(h2, in);
    }
    // rhs -= (c4 k2) f ; rhs += (c5 k2z) fz
    const double ar = DMUL(c4, k2r[l]), ai = DMUL(c4, k2i[l]);
    const double f_r = fr.p[0][e], f_i = fi.p[0][e];
    out[0] = __dsub_rn(out[0], __dsub_rn(DMUL(ar, f_r), DMUL(ai, f_i)));
    out[1] = __dsub_rn(out[1], DADD(DMUL(ar, f_i), DMUL(ai, f_r)));
    const double br = DMUL(c5, k2zr[l]), bi = DMUL(c5, k2zi[l]);
    const double z_r = fr.p[6][e], z_i = fi.p[6][e];
    out[0] = DADD(out[0], __dsub_rn(DMUL(br, z_r), DMUL(bi, z_i)));
    out[1] = DADD(out[1], DADD(DMUL(br, z_i), DMUL(bi, z_r)));
    Fr[e] = out[0];
    Fi[e] = out[1];
  }
}

__global__ void rhs_convdiff_z_kernel(Fields7 fr, Fields7 fi, double hx2, double hy2,
                                      double hz2, double gr, double gi, long long n,
                                      double* __restrict__ Fr, double* __restrict__ Fi) {
  const double a = __ddiv_rn(hx2, 12.0), b = __ddiv_rn(hy2, 12.0), c = __ddiv_rn(hz2, 12.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    // fields: f, fxx, fyy, fz, fzz
    const double zr = fr.p[3][e], zi = fi.p[3][e];
    const double gzr = DADD(__dsub_rn(DMUL(gr, zr), DMUL(gi, zi)), fr.p[4][e]);
    const double gzi = DADD(DADD(DMUL(gr, zi), DMUL(gi, zr)), fi.p[4][e]);
    double inr = DADD(fr.p[0][e], DMUL(a, fr.p[1][e]));
    double ini = DADD(fi.p[0][e], DMUL(a, fi.p[1][e]));
    inr = DADD(inr, DMUL(b, fr.p[2][e]));
    ini = DADD(ini, DMUL(b, fi.p[2][e]));
    inr = DADD(inr, DMUL(c, gzr));
    ini = DADD(ini, DMUL(c, gzi));
    Fr[e] = DMUL(hz2, inr);
    Fi[e] = DMUL(hz2, ini);
  }
}

// 27-point operator on a closed box (assembly.py:229-244). Raw weights
// (a, b, c, d) per level and offset, in the reference's term order:
// for dl in (-1, 0, 1): for (di, dj) in _PLANE_OFFSETS (assembly.py:20-25).
__constant__ int c_off_di[9] = {-1, 1, -1, 1, -1, 1, 0, 0, 0};
__constant__ int c_off_dj[9] = {-1, -1, 1, 1, 0, 0, -1, 1, 0};
__constant__ int c_off_w[9] = {0, 0, 0, 0, 1, 1, 2, 2, 3};  // a a a a b b c c d

__device__ __forceinline__ double apply27_point(const double* __restrict__ ext,
                                                const double* __restrict__ raw, int i, int j,
                                                int l, long long X, long long XY,
                                                uint32_t mask) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const long long zb = (long long)(l + k) * XY;  // level l + (k-1), closed index +1
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      if (mask & (1u << (k * 9 + o))) {
        const double wgt = __ldg(&raw[(long long)l * 12 + k * 4 + c_off_w[o]]);
        const double v = __ldg(&ext[zb + (long long)(j + 1 + c_off_dj[o]) * X + (i + 1 + c_off_di[o])]);
        acc = DADD(acc, DMUL(wgt, v));
      }
    }
  }
  return acc;
}

// mode 0: out = A ext; mode 1: out = rhs - A ext (fold_dirichlet, assembly.py:258-274)
__global__ void apply27_kernel(const double* __restrict__ ext, const double* __restrict__ rhs,
                               double* __restrict__ out, const double* __restrict__ raw, int nx,
                               int ny, int nz, uint32_t mask, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y, l = blockIdx.z;
  if (i >= nx) return;
  const long long X = nx + 2, XY = (long long)(nx + 2) * (ny + 2);
  const double v = apply27_point(ext, raw, i, j, l, X, XY, mask);
  const long long o = ((long long)l * ny + j) * nx + i;
  out[o] = mode == 0 ? v : __dsub_rn(rhs[o], v);
}

// The 27-point operator marching up the levels (tuning key 20 > 0): a thread owns
// column (i, j) and keeps the three 3 x 3 planes around it in registers, so each
// level costs the nine values of one new plane instead of 27 gathers; the sum
// runs in apply27_point's order (k, then the offsets), bit for bit.
template <int TX, int TY>
__global__ void __launch_bounds__(TX * TY) apply27_march_kernel(
    const double* __restrict__ ext, const double* __restrict__ rhs, double* __restrict__ out,
    const double* __restrict__ raw, int nx, int ny, int nz, uint32_t mask, int mode, int lz) {
  const int i = blockIdx.x * TX + threadIdx.x % TX, j = blockIdx.y * TY + threadIdx.x / TX;
  if (i >= nx || j >= ny) return;
  const int l0 = blockIdx.z * lz, l1 = min(nz, l0 + lz);
  const long long X = nx + 2, XY = X * (ny + 2);
  const long long col = (long long)(j + 1) * X + (i + 1);
  // the offset tables as compile-time constants (registers, no constant-bank loads)
  constexpr int DI[9] = {-1, 1, -1, 1, -1, 1, 0, 0, 0};
  constexpr int DJ[9] = {-1, -1, 1, 1, 0, 0, -1, 1, 0};
  constexpr int WI[9] = {0, 0, 0, 0, 1, 1, 2, 2, 3};
  double pl[3][9];
  auto load_plane = [&](int L, double* d) {  // closed plane L around the column
    const long long b = (long long)L * XY + col;
#pragma unroll
    for (int o = 0; o < 9; ++o) d[o] = __ldg(&ext[b + (long long)DJ[o] * X + DI[o]]);
  };
  load_plane(l0, pl[0]);
  load_plane(l0 + 1, pl[1]);
  for (int l = l0; l < l1; ++l) {
    load_plane(l + 2, pl[2]);
    double w[12];  // this level's weights (the same for every thread: broadcast loads)
#pragma unroll
    for (int q = 0; q < 12; ++q) w[q] = __ldg(&raw[(long long)l * 12 + q]);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int o = 0; o < 9; ++o)
        if (mask & (1u << (k * 9 + o))) acc = DADD(acc, DMUL(w[k * 4 + WI[o]], pl[k][o]));
    const long long oo = ((long long)l * ny + j) * nx + i;
    out[oo] = mode == 0 ? acc : __dsub_rn(rhs[oo], acc);
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      pl[0][o] = pl[1][o];
      pl[1][o] = pl[2][o];
    }
  }
}

// Residual sum of squares with a zero boundary: u is interior-only, so the
// neighbour fetch is bounds-checked instead of padded (assembly.py:277-289).
__global__ void residual_sq_kernel(const double* __restrict__ u, const double* __restrict__ F,
                                   const double* __restrict__ raw, int nx, int ny, int nz,
                                   uint32_t mask, double* __restrict__ partial) {
  __shared__ double red[256 / 32];
  const long long n = (long long)nx * ny * nz;
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const int j = (int)((e / nx) % ny);
    const int l = (int)(e / ((long long)nx * ny));
    double acc = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int ll = l + k - 1;
      for (int o = 0; o < 9; ++o) {
        if (!(mask & (1u << (k * 9 + o)))) continue;
        const int ii = i + c_off_di[o], jj = j + c_off_dj[o];
        double v = 0.0;
        if (ll >= 0 && ll < nz && jj >= 0 && jj < ny && ii >= 0 && ii < nx)
          v = u[((long long)ll * ny + jj) * nx + ii];
        acc = DADD(acc, DMUL(raw[(long long)l * 12 + k * 4 + c_off_w[o]], v));
      }
    }
    const double r = acc - F[e];
    s = fma(r, r, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 256 / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// The residual, marching: 148 x 8 persistent CTAs (the partial-sum count of
// hfb_residual_partials) walk 64 x 4 column tiles of lz levels; a thread keeps
// the three 3 x 3 planes of u around its column in registers (zero outside the
// interior) and the level's weights, and sums the terms in residual_sq_kernel's
// order. Only the order of the final sum of squares differs.
template <int TX, int TY>
__global__ void __launch_bounds__(TX * TY) residual_sq_march_kernel(
    const double* __restrict__ u, const double* __restrict__ F, const double* __restrict__ raw,
    int nx, int ny, int nz, uint32_t mask, double* __restrict__ partial, int lz) {
  constexpr int DI[9] = {-1, 1, -1, 1, -1, 1, 0, 0, 0};
  constexpr int DJ[9] = {-1, -1, 1, 1, 0, 0, -1, 1, 0};
  constexpr int WI[9] = {0, 0, 0, 0, 1, 1, 2, 2, 3};
  __shared__ double red[TX * TY / 32];
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int gx = (nx + TX - 1) / TX, gy = (ny + TY - 1) / TY, gz = (nz + lz - 1) / lz;
  const long long items = (long long)gx * gy * gz;
  const long long XY = (long long)nx * ny;
  double s = 0.0;
  for (long long it = blockIdx.x; it < items; it += gridDim.x) {
    const int bx = (int)(it % gx), by = (int)((it / gx) % gy), bz = (int)(it / ((long long)gx * gy));
    const int i = bx * TX + tx, j = by * TY + ty;
    if (i >= nx || j >= ny) continue;
    const int l0 = bz * lz, l1 = min(nz, l0 + lz);
    auto load_plane = [&](int L, double* d) {
#pragma unroll
      for (int o = 0; o < 9; ++o) {
        const int ii = i + DI[o], jj = j + DJ[o];
        d[o] = (L >= 0 && L < nz && ii >= 0 && ii < nx && jj >= 0 && jj < ny)
                   ? __ldg(&u[(long long)L * XY + (long long)jj * nx + ii])
                   : 0.0;
      }
    };
    double pl[3][9];
    load_plane(l0 - 1, pl[0]);
    load_plane(l0, pl[1]);
    for (int l = l0; l < l1; ++l) {
      load_plane(l + 1, pl[2]);
      double w[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) w[q] = __ldg(&raw[(long long)l * 12 + q]);
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int o = 0; o < 9; ++o)
          if (mask & (1u << (k * 9 + o))) acc = DADD(acc, DMUL(w[k * 4 + WI[o]], pl[k][o]));
      const double r = acc - F[(long long)l * XY + (long long)j * nx + i];
      s = fma(r, r, s);
#pragma unroll
      for (int o = 0; o < 9; ++o) {
        pl[0][o] = pl[1][o];
        pl[1][o] = pl[2][o];
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < TX * TY / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// The 27-point operator streamed plane by plane (tuning key 24 > 0: levels per
// CTA). A warp owns 32 consecutive x-points of RJ consecutive rows; every closed
// plane P is loaded once per warp (rows j0-1 .. j0+RJ, columns i-1 .. i+1, 3 (RJ+2)
// loads for RJ points instead of 9 per point) and immediately contributes its
// k = 0, 1, 2 terms to the running sums of output levels P, P-1 and P-2. Plane P
// arrives after P-1, so each output still adds (k = 0 terms, k = 1, k = 2) in
// the reference's order (assembly.py:229-244), every term DMUL then DADD: bit for
// bit apply27_point. Three sums per point live in registers instead of the
// 27-value window of the marching kernels.
//   KIND 0: out = A ext;  KIND 1: out = rhs - A ext (ext closed, (nz+2, ny+2, nx+2))
//   KIND 2: sum of (A u - F)^2 with u interior and zero outside (assembly.py:277-289);
//           one partial per CTA (hfb_residual_partials)
template <int RJ, int KIND>
__global__ void __launch_bounds__(256, (RJ <= 2 ? 3 : 2)) s27_stream_kernel(
    const double* __restrict__ src, const double* __restrict__ rhs, double* __restrict__ out,
    const double* __restrict__ raw, int nx, int ny, int nz, uint32_t mask, int lz,
    double* __restrict__ partial) {
  constexpr int DI[9] = {-1, 1, -1, 1, -1, 1, 0, 0, 0};
  constexpr int DJ[9] = {-1, -1, 1, 1, 0, 0, -1, 1, 0};
  constexpr int WI[9] = {0, 0, 0, 0, 1, 1, 2, 2, 3};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int j0 = (blockIdx.y * 8 + warp) * RJ;
  const int l0 = blockIdx.z * lz, l1 = min(nz, l0 + lz);
  const long long X = KIND == 2 ? nx : nx + 2;
  const long long XY = X * (KIND == 2 ? ny : ny + 2);
  // per-thread column offsets (clamped into the array: lanes past nx compute
  // garbage they never store)
  long long coff[3];
  bool cok[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int ii = i - 1 + c;  // interior column
    if constexpr (KIND == 2) {
      cok[c] = ii >= 0 && ii < nx;
      coff[c] = min(max(ii, 0), nx - 1);
    } else {
      cok[c] = true;
      coff[c] = min(ii + 1, nx + 1);
    }
  }
  double a0[RJ], a1[RJ], a2[RJ];  // running sums of output levels P-2, P-1, P
#pragma unroll
  for (int q = 0; q < RJ; ++q) a0[q] = a1[q] = 0.0;
  double ssq = 0.0;
  for (int P = l0; P <= l1 + 1; ++P) {  // closed plane P = interior plane P - 1
    double v[RJ + 2][3];
    const int ql = P - 1;
    const bool pok = KIND != 2 || (ql >= 0 && ql < nz);
#pragma unroll
    for (int r = 0; r < RJ + 2; ++r) {
      const int jr = j0 - 1 + r;  // interior row
      long long rb;
      bool rok;
      if constexpr (KIND == 2) {
        rok = pok && jr >= 0 && jr < ny;
        rb = (long long)min(max(ql, 0), nz - 1) * XY + (long long)min(max(jr, 0), ny - 1) * X;
      } else {
        rok = true;
        rb = (long long)P * XY + (long long)min(jr + 1, ny + 1) * X;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) v[r][c] = (rok && cok[c]) ? __ldg(src + rb + coff[c]) : 0.0;
    }
    // weights of the three output levels this plane serves (clamped indices for
    // levels outside [l0, l1): their sums are never stored)
    const double* w0 = raw + (long long)min(P, nz - 1) * 12;                   // level P, k = 0
    const double* w1 = raw + (long long)min(max(P - 1, 0), nz - 1) * 12 + 4;   // level P-1, k = 1
    const double* w2 = raw + (long long)max(P - 2, 0) * 12 + 8;                // level P-2, k = 2
    double wk0[4], wk1[4], wk2[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      wk0[q] = __ldg(w0 + q);
      wk1[q] = __ldg(w1 + q);
      wk2[q] = __ldg(w2 + q);
    }
#pragma unroll
    for (int q = 0; q < RJ; ++q) {
      double t0 = 0.0, t1 = a1[q], t2 = a0[q];
#pragma unroll
      for (int o = 0; o < 9; ++o) {
        const double x = v[q + 1 + DJ[o]][1 + DI[o]];
        if (mask & (1u << o)) t0 = DADD(t0, DMUL(wk0[WI[o]], x));
      }
#pragma unroll
      for (int o = 0; o < 9; ++o) {
        const double x = v[q + 1 + DJ[o]][1 + DI[o]];
        if (mask & (1u << (9 + o))) t1 = DADD(t1, DMUL(wk1[WI[o]], x));
      }
#pragma unroll
      for (int o = 0; o < 9; ++o) {
        const double x = v[q + 1 + DJ[o]][1 + DI[o]];
        if (mask & (1u << (18 + o))) t2 = DADD(t2, DMUL(wk2[WI[o]], x));
      }
      // t2 completes output level P - 2
      const int L = P - 2, j = j0 + q;
      if (L >= l0 && i < nx && j < ny) {
        const long long oo = ((long long)L * ny + j) * nx + i;
        if constexpr (KIND == 0) out[oo] = t2;
        if constexpr (KIND == 1) out[oo] = __dsub_rn(__ldg(rhs + oo), t2);
        if constexpr (KIND == 2) {
          const double rr = t2 - __ldg(rhs + oo);
          ssq = fma(rr, rr, ssq);
        }
      }
      a0[q] = t1;
      a1[q] = t0;
    }
  }
  if constexpr (KIND == 2) {
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) ssq += __shfl_down_sync(0xffffffffu, ssq, o);
    if (lane == 0) red[warp] = ssq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      partial[blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z)] = t;
    }
  }
}

// The same streamed 27-point sums with the planes staged in shared memory
// (tuning key 27, default): a CTA owns a 32 x 32 output tile and marches
// lz levels; the 34 x 34 input tile of each plane (halo included) arrives by
// 8-byte cp.async four planes ahead of the arithmetic (zero-filled outside the
// array, which is the residual's zero boundary), so the FP64 pipe no longer
// waits on the loads that head every plane of s27_stream_kernel. rhs / F of
// the level being completed are prefetched into registers one plane ahead.
// Same term order, same bits.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}
// the same with the destination as a shared-window address
__device__ __forceinline__ void cp_async8_s(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kT27NS = 4;                   // plane stages
constexpr int kT27Pitch = 36;               // doubles per staged row (34 used)
constexpr int kT27Stage = 34 * kT27Pitch;   // doubles per stage

// CM != 0: the term mask as a compile-time constant (the full 27-term mask of
// the 6th-order and general tables, the 19-term mask of the 4th-order and cd4
// tables): the per-term tests fold away (with a runtime mask they cost more
// instructions than the arithmetic).
constexpr uint32_t kMask27 = 0x7FFFFFFu, kMask19 = 0x7C3FFF0u;

template <int KIND, uint32_t CM>
__global__ void __launch_bounds__(256, 2) s27_tile_kernel(
    const double* __restrict__ src, const double* __restrict__ rhs, double* __restrict__ out,
    const double* __restrict__ raw, int nx, int ny, int nz, uint32_t mask_rt, int lz,
    double* __restrict__ partial) {
  const uint32_t mask = CM ? CM : mask_rt;
  constexpr int RJ = 4, NS = kT27NS, PT = kT27Pitch;
  constexpr int DI[9] = {-1, 1, -1, 1, -1, 1, 0, 0, 0};
  constexpr int DJ[9] = {-1, -1, 1, 1, 0, 0, -1, 1, 0};
  constexpr int WI[9] = {0, 0, 0, 0, 1, 1, 2, 2, 3};
  extern __shared__ __align__(16) double smt[];
  // this CTA's levels' raw weights, after the plane stages and (KIND != 0)
  // the rhs stages
  double* wsm = smt + NS * kT27Stage + (KIND != 0 ? NS * 1024 : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  const int l0 = blockIdx.z * lz, l1 = min(nz, l0 + lz);
  const int i = x0 + lane, jw = y0 + warp * RJ;
  // weights of levels l0 - 2 .. l1 + 1 with the out-of-range levels replicated
  // from the nearest level of the CTA: plane P then reads its three weight rows
  // (levels P - 2, P - 1, P, clamped as before) at fixed offsets from one pointer
  for (int e = threadIdx.x; e < (l1 - l0 + 4) * 12; e += 256) {
    const int lev = min(max(l0 - 2 + e / 12, l0), l1 - 1);
    wsm[e] = __ldg(raw + lev * 12LL + e % 12);
  }
  // this thread's (at most 5) elements of the 34 x 34 input tile: byte offset
  // in a stage, offset from the plane base (coordinates clamped into the array,
  // so every copy reads a valid address) and whether the element lies in the
  // array (the residual also checks the plane); out-of-array elements are
  // zero-filled by the copy (source size 0)
  constexpr int NE = (34 * 34 + 255) / 256;
  int soff[NE], goff[NE];
  unsigned eok = 0;
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    const int e = threadIdx.x + 256 * q;
    const int r = e / 34, c = e - r * 34;
    const int gy = y0 - 1 + r, gx = x0 - 1 + c;  // interior coordinates
    soff[q] = e < 34 * 34 ? 8 * (r * PT + c) : -1;
    bool ok;
    if constexpr (KIND == 2) {
      ok = gy >= 0 && gy < ny && gx >= 0 && gx < nx;
      goff[q] = min(max(gy, 0), ny - 1) * nx + min(max(gx, 0), nx - 1);
    } else {
      ok = gy + 1 <= ny + 1 && gx + 1 <= nx + 1;
      goff[q] = min(gy + 1, ny + 1) * (nx + 2) + min(gx + 1, nx + 1);
    }
    eok |= (ok && e < 34 * 34) ? 1u << q : 0u;
  }
  const long long pstride = KIND == 2 ? (long long)nx * ny : (long long)(nx + 2) * (ny + 2);
  const uint32_t sbase = smem_u32(smt);
  // rhs / F of output level P - 2 rides with plane P: this thread's own 4 values
  const uint32_t rbase = smem_u32(smt + NS * kT27Stage) + 8 * (warp * RJ * 32 + lane);
  const bool icol = i < nx;
  // the next plane to load (a running pointer: one 64-bit add per plane instead
  // of a 64-bit product); the residual's planes outside the array are never read
  // (zero-filled copies of size 0 from a valid address)
  const double* nextp = src + (long long)(KIND == 2 ? l0 - 1 : l0) * pstride;
  // rhs / F rows of level P - 2 and the output rows: plane stride of the interior
  // arrays, this thread's row offsets (clamped into the plane)
  const long long ostep = (long long)ny * nx;
  const double* nextr = KIND == 0 ? nullptr : rhs + (long long)(l0 - 2) * ostep + min(i, nx - 1);
  int roff[RJ];
#pragma unroll
  for (int q = 0; q < RJ; ++q) roff[q] = min(jw + q, ny - 1) * nx;
  auto load_plane = [&](int P, int st) {
    const uint32_t dst = sbase + st * (kT27Stage * 8);
    const bool pok = KIND != 2 || (P >= 1 && P <= nz);
    const double* base = pok ? nextp : src;
    nextp += pstride;
#pragma unroll
    for (int q = 0; q < NE; ++q) {
      if (soff[q] < 0) continue;
      cp_async8_s(dst + soff[q], base + goff[q], (pok && ((eok >> q) & 1u)) ? 8 : 0);
    }
    if constexpr (KIND != 0) {
      const int L = P - 2;
      const bool lok = L >= l0 && L < l1 && icol;
      const double* rb = lok ? nextr : rhs;  // level L's rows (a running pointer)
      nextr += ostep;
      const uint32_t rd = rbase + st * (1024 * 8);
#pragma unroll
      for (int q = 0; q < RJ; ++q)
        cp_async8_s(rd + q * 32 * 8, rb + roff[q], (lok && jw + q < ny) ? 8 : 0);
    }
  };
  const int Pend = l1 + 1;  // planes l0 .. l1 + 1 serve levels l0 .. l1 - 1
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    if (l0 + q <= Pend) load_plane(l0 + q, q);
    cp_async_commit();
  }
  double a0[RJ], a1[RJ];
#pragma unroll
  for (int q = 0; q < RJ; ++q) a0[q] = a1[q] = 0.0;
  double ssq = 0.0;
  bool rowok[RJ];
#pragma unroll
  for (int q = 0; q < RJ; ++q) rowok[q] = icol && jw + q < ny;
  // output row of level L = P - 2, this thread's column: advanced by a plane per step
  double* op = KIND == 2 ? nullptr : out + ((long long)l0 * ny + jw) * nx + i - 2 * ostep;
  auto plane_step = [&](int P) {
    cp_async_wait<NS - 2>();
    __syncthreads();  // plane P staged for everyone; stage (P - 1) free
    if (P + NS - 1 <= Pend) load_plane(P + NS - 1, (P + NS - 1 - l0) % NS);
    cp_async_commit();
    const double* pl = smt + ((P - l0) % NS) * kT27Stage + warp * RJ * PT + lane;
    const double* rl = smt + NS * kT27Stage + ((P - l0) % NS) * 1024 + warp * RJ * 32 + lane;
    const double* wp = wsm + (P - l0) * 12;  // the row of level P - 2 (replicated table)
    const double* w0 = wp + 24;              // level P, k = 0
    const double* w1 = wp + 12 + 4;          // level P-1, k = 1
    const double* w2 = wp + 8;               // level P-2, k = 2
    double wk0[4], wk1[4], wk2[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      wk0[q] = w0[q];
      wk1[q] = w1[q];
      wk2[q] = w2[q];
    }
    const int L = P - 2;
    double* orow = op;  // out + ((L ny) + jw) nx + i: a running pointer (valid once L >= l0)
    if constexpr (KIND != 2) op += ostep;
#pragma unroll
    for (int q = 0; q < RJ; ++q) {
      double v[9];
#pragma unroll
      for (int o = 0; o < 9; ++o) v[o] = pl[(q + 1 + DJ[o]) * PT + 1 + DI[o]];
      double t0 = 0.0, t1 = a1[q], t2 = a0[q];
#pragma unroll
      for (int o = 0; o < 9; ++o)
        if (mask & (1u << o)) t0 = DADD(t0, DMUL(wk0[WI[o]], v[o]));
#pragma unroll
      for (int o = 0; o < 9; ++o)
        if (mask & (1u << (9 + o))) t1 = DADD(t1, DMUL(wk1[WI[o]], v[o]));
#pragma unroll
      for (int o = 0; o < 9; ++o)
        if (mask & (1u << (18 + o))) t2 = DADD(t2, DMUL(wk2[WI[o]], v[o]));
      const int j = jw + q;
      if constexpr (KIND == 0) {
        // (row pointer once per plane, row tests once per kernel: fewer
        // registers for the twice-unrolled apply loop)
        if (L >= l0 && rowok[q]) orow[q * nx] = t2;
      } else if (L >= l0 && i < nx && j < ny) {
        if constexpr (KIND == 1) orow[q * nx] = __dsub_rn(rl[q * 32], t2);
        if constexpr (KIND == 2) {
          const double rr = t2 - rl[q * 32];
          ssq = fma(rr, rr, ssq);
        }
      }
      a0[q] = t1;
      a1[q] = t0;
    }
  };
  // the plane loop is unrolled twice (the (a0, a1) <- (t1, t0) rotation then
  // needs no register moves); with the running pointers all three kinds fit
  // the 128-register budget without spills (fold 5.4 -> 5.1-5.2 ms, residual
  // 4.75 -> 4.61 ms at 1023^3)
#ifndef HFB_S27_UNROLL2
#define HFB_S27_UNROLL2 7  // bit 0: apply, bit 1: fold, bit 2: residual (all: no spills since the running pointers)
#endif
  if constexpr (((HFB_S27_UNROLL2) >> KIND) & 1) {
#pragma unroll 2
    for (int P = l0; P <= Pend; ++P) plane_step(P);
  } else {
    for (int P = l0; P <= Pend; ++P) plane_step(P);
  }
  cp_async_wait<0>();
  if constexpr (KIND == 2) {
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) ssq += __shfl_down_sync(0xffffffffu, ssq, o);
    if (lane == 0) red[warp] = ssq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      partial[blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z)] = t;
    }
  }
}

constexpr int kS27ResLz = 32;  // levels per CTA of the streamed residual (fixes the partial count)

// rows per warp of the streamed 27-point kernels (tuning key 25: 2 or 4)
static int s27_rj() { return tuning(25) == 2 ? 2 : 4; }

static dim3 s27_grid(const hfb_plan* p, int lz, int rj) {
  return dim3((p->nx + 31) / 32, (p->ny + 8 * rj - 1) / (8 * rj), (p->nz + lz - 1) / lz);
}

// levels per CTA of the streamed kernels: at least enough to keep gridDim.z
// within its 65535 limit
static int s27_lz(const hfb_plan* p, int lz) { return std::max(lz, (p->nz + 65534) / 65535); }

template <int KIND>
static int s27_launch(const hfb_plan* p, int lz, const double* src, const double* rhs,
                      double* out, uint32_t mask, double* partial, cudaStream_t st) {
  const int rj = s27_rj();
  const double* raw = p->coef + 12LL * p->nz;
  if (tuning(27)) {  // shared-memory staged planes (32 x 32 tiles = the rj = 4 grid)
    const size_t sm = sizeof(double) * ((size_t)kT27NS * (kT27Stage + (KIND ? 1024 : 0)) +
                                        12 * ((size_t)lz + 4));
    auto kern = mask == kMask27 ? s27_tile_kernel<KIND, kMask27>
                : mask == kMask19 ? s27_tile_kernel<KIND, kMask19>
                                  : s27_tile_kernel<KIND, 0>;
    HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<s27_grid(p, lz, 4), 256, sm, st>>>(src, rhs, out, raw, p->nx, p->ny, p->nz, mask, lz,
                                              partial);
    return HFB_OK;
  }
  if (rj == 2)
    s27_stream_kernel<2, KIND><<<s27_grid(p, lz, 2), 256, 0, st>>>(
        src, rhs, out, raw, p->nx, p->ny, p->nz, mask, lz, partial);
  else
    s27_stream_kernel<4, KIND><<<s27_grid(p, lz, 4), 256, 0, st>>>(
        src, rhs, out, raw, p->nx, p->ny, p->nz, mask, lz, partial);
  return HFB_OK;
}

// Complex weights (complex k(z)): out = A ext or rhs - A ext with complex
// arithmetic, each term w * v = (wr vr - wi vi, wr vi + wi vr) added in the
// reference's order (assembly.py:229-244 on complex128).
__global__ void apply27_z_kernel(const double* __restrict__ er, const double* __restrict__ ei,
                                 const double* __restrict__ rr, const double* __restrict__ ri,
                                 double* __restrict__ outr, double* __restrict__ outi,
                                 const double* __restrict__ rawr, const double* __restrict__ rawi,
                                 int nx, int ny, int nz, uint32_t mask, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y, l = blockIdx.z;
  if (i >= nx) return;
  const long long X = nx + 2, XY = (long long)(nx + 2) * (ny + 2);
  double ar = 0.0, ai = 0.0;
  for (int k = 0; k < 3; ++k) {
    const long long zb = (long long)(l + k) * XY;
    for (int o = 0; o < 9; ++o) {
      if (!(mask & (1u << (k * 9 + o)))) continue;
      const long long w = (long long)l * 12 + k * 4 + c_off_w[o];
      const double wr = __ldg(&rawr[w]), wi = __ldg(&rawi[w]);
      const long long e = zb + (long long)(j + 1 + c_off_dj[o]) * X + (i + 1 + c_off_di[o]);
      const double vr = __ldg(&er[e]), vi = __ldg(&ei[e]);
      ar = DADD(ar, __dsub_rn(DMUL(wr, vr), DMUL(wi, vi)));
      ai = DADD(ai, DADD(DMUL(wr, vi), DMUL(wi, vr)));
    }
  }
  const long long o = ((long long)l * ny + j) * nx + i;
  outr[o] = mode == 0 ? ar : __dsub_rn(rr[o], ar);
  outi[o] = mode == 0 ? ai : __dsub_rn(ri[o], ai);
}

// |A u - F|^2 partial sums (complex), zero boundary, as residual_sq_kernel.
__global__ void residual_sq_z_kernel(const double* __restrict__ ur, const double* __restrict__ ui,
                                     const double* __restrict__ Fr, const double* __restrict__ Fi,
                                     const double* __restrict__ rawr,
                                     const double* __restrict__ rawi, int nx, int ny, int nz,
                                     uint32_t mask, double* __restrict__ partial) {
  __shared__ double red[256 / 32];
  const long long n = (long long)nx * ny * nz;
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const int j = (int)((e / nx) % ny);
    const int l = (int)(e / ((long long)nx * ny));
    double ar = 0.0, ai = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int ll = l + k - 1;
      for (int o = 0; o < 9; ++o) {
        if (!(mask & (1u << (k * 9 + o)))) continue;
        const int ii = i + c_off_di[o], jj = j + c_off_dj[o];
        double vr = 0.0, vi = 0.0;
        if (ll >= 0 && ll < nz && jj >= 0 && jj < ny && ii >= 0 && ii < nx) {
          const long long q = ((long long)ll * ny + jj) * nx + ii;
          vr = ur[q];
          vi = ui[q];
        }
        const long long w = (long long)l * 12 + k * 4 + c_off_w[o];
        ar = DADD(ar, __dsub_rn(DMUL(rawr[w], vr), DMUL(rawi[w], vi)));
        ai = DADD(ai, DADD(DMUL(rawr[w], vi), DMUL(rawi[w], vr)));
      }
    }
    const double dr = ar - Fr[e], di = ai - Fi[e];
    s = fma(dr, dr, fma(di, di, s));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 256 / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

// slab (kpz, ny, nx) -> send blocks (kpz, kpy(q), nx), ascending q
__global__ void pack_yblocks_kernel(const double* __restrict__ slab, double* __restrict__ send,
                                    int kpz, int ny, int nx, const int* __restrict__ ys,
                                    int parts) {
  const long long total = (long long)kpz * ny * nx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const int j = (int)((e / nx) % ny);
    const int l = (int)(e / ((long long)nx * ny));
    int q = 0;
    while (q + 1 < parts && j >= ys[q + 1]) ++q;
    const int y0 = ys[q], kpy = ys[q + 1] - ys[q];
    const long long base = (long long)kpz * y0 * nx;  // blocks before q
    send[base + ((long long)l * kpy + (j - y0)) * nx + i] = slab[e];
  }
}

__global__ void unpack_yblocks_kernel(const double* __restrict__ recv, double* __restrict__ slab,
                                      int kpz, int ny, int nx, const int* __restrict__ ys,
                                      int parts) {
  const long long total = (long long)kpz * ny * nx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const int j = (int)((e / nx) % ny);
    const int l = (int)(e / ((long long)nx * ny));
    int q = 0;
    while (q + 1 < parts && j >= ys[q + 1]) ++q;
    const int y0 = ys[q], kpy = ys[q + 1] - ys[q];
    const long long base = (long long)kpz * y0 * nx;
    slab[e] = recv[base + ((long long)l * kpy + (j - y0)) * nx + i];
  }
}

}  // namespace hfb

// ------------------------------------------------------------------ C-ABI
using namespace hfb;

static unsigned grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b > 148LL * 64) b = 148LL * 64;
  if (b < 1) b = 1;
  return (unsigned)b;
}

extern "C" int hfb_rhs_fourth(hfb_plan* p, const double* f, double* F, double hz2,
                              void* stream) {
  const NvtxRange nvtx_("hfb_rhs_fourth");
  if (!p || !f || !F) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  const int v = tuning(20);
  if (v > 0) {  // marching columns (v = levels per CTA)
    // 64 x 4 columns, v levels per CTA (measured: 3.45 ms at v = 32 against
    // 4.33 ms for the per-point gathers at 1023^3, tools/stencil_rate.py)
    constexpr int TX = 64, TY = 4;
    dim3 grid((p->nx + TX - 1) / TX, (p->ny + TY - 1) / TY, (p->nz + v - 1) / v);
    rhs_fourth_march_kernel<TX, TY><<<grid, TX * TY, 0, (cudaStream_t)stream>>>(
        f, F, p->nx, p->ny, p->nz, hz2, v);
  } else {
    dim3 grid((p->nx + 127) / 128, p->ny, p->nz);
    rhs_fourth_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(f, F, p->nx, p->ny, p->nz, hz2);
  }
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_rhs_second(hfb_plan* p, const double* f, double* F, double hz2,
                              void* stream) {
  if (!p || !f || !F) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  const long long n = (long long)p->nx * p->ny * p->nz;
  rhs_second_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(f, F, n, hz2);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_rhs_sixth(hfb_plan* p, const double* f, const double* lap, const double* d4,
                             const double* fxxyy, const double* fxxzz, const double* fyyzz,
                             const double* fz, const double* k2, const double* k2z, double h2,
                             double* F, void* stream) {
  if (!p || !f || !lap || !d4 || !fxxyy || !fxxzz || !fyyzz || !fz || !k2 || !k2z || !F)
    return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  const long long plane = (long long)p->nx * p->ny, n = plane * p->nz;
  rhs_sixth_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      f, lap, d4, fxxyy, fxxzz, fyyzz, fz, k2, k2z, h2, plane, n, F);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_rhs_convdiff(hfb_plan* p, const double* f, const double* fxx,
                                const double* fyy, const double* fz, const double* fzz,
                                double hx2, double hy2, double hz2, double gamma, double* F,
                                void* stream) {
  if (!p || !f || !fxx || !fyy || !fz || !fzz || !F) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  const long long n = (long long)p->nx * p->ny * p->nz;
  rhs_convdiff_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      f, fxx, fyy, fz, fzz, hx2, hy2, hz2, gamma, n, F);
  HFB_LAUNCHED();
  return HFB_OK;
}

// raw table pointer: the plan keeps the scaled (4a,2b,2c,d) copy for the
// Thomas sweep and the raw (a,b,c,d) copy right after it.
extern "C" int hfb_apply27(hfb_plan* p, const double* ext, const double* rhs, double* out,
                           uint32_t mask, int mode, void* stream) {
  const NvtxRange nvtx_("hfb_apply27");
  if (!p || !ext || !out || (mode == 1 && !rhs)) return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  HFB_CUDA(cudaSetDevice(p->device));
  const int lz = tuning(20), ls = tuning(24);
  if (ls > 0) {
    const int rc = mode == 0 ? s27_launch<0>(p, s27_lz(p, ls), ext, rhs, out, mask, nullptr,
                                             (cudaStream_t)stream)
                             : s27_launch<1>(p, s27_lz(p, ls), ext, rhs, out, mask, nullptr,
                                             (cudaStream_t)stream);
    if (rc) return rc;
  } else if (lz > 0) {
    constexpr int TX = 64, TY = 4;
    dim3 grid((p->nx + TX - 1) / TX, (p->ny + TY - 1) / TY, (p->nz + lz - 1) / lz);
    apply27_march_kernel<TX, TY><<<grid, TX * TY, 0, (cudaStream_t)stream>>>(
        ext, rhs, out, p->coef + 12LL * p->nz, p->nx, p->ny, p->nz, mask, mode, lz);
  } else {
    dim3 grid((p->nx + 127) / 128, p->ny, p->nz);
    apply27_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(ext, rhs, out, p->coef + 12LL * p->nz,
                                                           p->nx, p->ny, p->nz, mask, mode);
  }
  HFB_LAUNCHED();
  return HFB_OK;
}

// One partial per CTA of the streamed residual (its tile count), at least the
// 148 x 8 persistent CTAs of the marching / gather / complex kernels.
extern "C" int hfb_residual_partials(const hfb_plan* p) {
  if (!p) return 148 * 8;
  const dim3 g = s27_grid(p, s27_lz(p, kS27ResLz), 2);  // the larger of the two tile counts
  const long long tiles = (long long)g.x * g.y * g.z;
  return (int)std::max<long long>(tiles, 148 * 8);
}

extern "C" int hfb_residual_sq(hfb_plan* p, const double* u, const double* F, double* partial,
                               uint32_t mask, void* stream) {
  const NvtxRange nvtx_("hfb_residual_sq");
  if (!p || !u || !F || !partial) return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  HFB_CUDA(cudaSetDevice(p->device));
  const int lz = tuning(20);
  const unsigned npart = (unsigned)hfb_residual_partials(p);
  if (tuning(24) > 0) {
    const int lr = s27_lz(p, kS27ResLz);
    const dim3 g = s27_grid(p, lr, tuning(27) ? 4 : s27_rj());
    const int rc = s27_launch<2>(p, lr, u, F, nullptr, mask, partial, (cudaStream_t)stream);
    if (rc) return rc;
    const unsigned used = g.x * g.y * g.z;
    if (npart > used)
      HFB_CUDA(cudaMemsetAsync(partial + used, 0, sizeof(double) * (npart - used),
                               (cudaStream_t)stream));
  } else if (lz > 0) {
    residual_sq_march_kernel<64, 4><<<npart, 256, 0, (cudaStream_t)stream>>>(
        u, F, p->coef + 12LL * p->nz, p->nx, p->ny, p->nz, mask, partial, lz);
  } else {
    residual_sq_kernel<<<npart, 256, 0, (cudaStream_t)stream>>>(
        u, F, p->coef + 12LL * p->nz, p->nx, p->ny, p->nz, mask, partial);
  }
  HFB_LAUNCHED();
  return HFB_OK;
}

static int upload_ystarts(hfb_plan* p, const int* ys, int parts, cudaStream_t st) {
  if (p->ystarts_cap < parts + 1) {
    if (p->ystarts) cudaFree(p->ystarts);
    p->ystarts = nullptr;
    HFB_CUDA(cudaMalloc(&p->ystarts, sizeof(int) * (parts + 1)));
    p->ystarts_cap = parts + 1;
  }
  HFB_CUDA(cudaMemcpyAsync(p->ystarts, ys, sizeof(int) * (parts + 1), cudaMemcpyHostToDevice, st));
  return HFB_OK;
}

extern "C" int hfb_pack_yblocks(hfb_plan* p, const double* slab, double* send, int kpz,
                                const int* ys, int parts, void* stream) {
  if (!p || !slab || !send || !ys || parts < 1 || kpz < 0) return HFB_ERR_ARGUMENT;
  if (ys[0] != 0 || ys[parts] != p->ny) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  int rc = upload_ystarts(p, ys, parts, (cudaStream_t)stream);
  if (rc) return rc;
  const long long n = (long long)kpz * p->ny * p->nx;
  if (n == 0) return HFB_OK;
  pack_yblocks_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      slab, send, kpz, p->ny, p->nx, p->ystarts, parts);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_unpack_yblocks(hfb_plan* p, const double* recv, double* slab, int kpz,
                                  const int* ys, int parts, void* stream) {
  if (!p || !slab || !recv || !ys || parts < 1 || kpz < 0) return HFB_ERR_ARGUMENT;
  if (ys[0] != 0 || ys[parts] != p->ny) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  int rc = upload_ystarts(p, ys, parts, (cudaStream_t)stream);
  if (rc) return rc;
  const long long n = (long long)kpz * p->ny * p->nx;
  if (n == 0) return HFB_OK;
  unpack_yblocks_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      recv, slab, kpz, p->ny, p->nx, p->ystarts, parts);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_apply27_z(hfb_plan* p, const double* ext_re, const double* ext_im,
                             const double* rhs_re, const double* rhs_im, double* out_re,
                             double* out_im, uint32_t mask, int mode, void* stream) {
  const NvtxRange nvtx_("hfb_apply27_z");
  if (!p || !ext_re || !ext_im || !out_re || !out_im) return HFB_ERR_ARGUMENT;
  if (mode == 1 && (!rhs_re || !rhs_im)) return HFB_ERR_ARGUMENT;
  if (!p->have_coef || !p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  HFB_CUDA(cudaSetDevice(p->device));
  dim3 grid((p->nx + 127) / 128, p->ny, p->nz);
  apply27_z_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(
      ext_re, ext_im, rhs_re, rhs_im, out_re, out_im, p->coef + 12LL * p->nz,
      p->coef_i + 12LL * p->nz, p->nx, p->ny, p->nz, mask, mode);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_residual_sq_z(hfb_plan* p, const double* u_re, const double* u_im,
                                 const double* rhs_re, const double* rhs_im, double* partial,
                                 uint32_t mask, void* stream) {
  const NvtxRange nvtx_("hfb_residual_sq_z");
  if (!p || !u_re || !u_im || !rhs_re || !rhs_im || !partial) return HFB_ERR_ARGUMENT;
  if (!p->have_coef || !p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  HFB_CUDA(cudaSetDevice(p->device));
  residual_sq_z_kernel<<<(unsigned)hfb_residual_partials(p), 256, 0, (cudaStream_t)stream>>>(
      u_re, u_im, rhs_re, rhs_im, p->coef + 12LL * p->nz, p->coef_i + 12LL * p->nz, p->nx,
      p->ny, p->nz, mask, partial);
  HFB_LAUNCHED();
  return HFB_OK;
}

// ---------------------------------------------------------------------------
// Mode-space exchange for the partitioned solve. A rank's
// transformed z-slab is padded mode rows (kpz, n_x, ldm); the block for rank q
// is (kpz, n_x, kp(q)) with kp(q) = its y-mode count rounded up to even, so the
// receiver's concatenation over senders is directly its y-slab of mode rows
// (n_z, n_x, kp) — 16-byte aligned rows for the TMA z-solve, no unpack.
namespace {
__device__ __forceinline__ int owner_of(const int* ys, int parts, int m, long long& base,
                                        int& kp, long long blk_rows) {
  base = 0;
  int q = 0;
  for (;; ++q) {
    kp = (ys[q + 1] - ys[q] + 1) & ~1;
    if (q == parts - 1 || m < ys[q + 1]) break;
    base += blk_rows * kp;
  }
  return q;
}
}  // namespace

__global__ void pack_modes_kernel(const double* __restrict__ modes, double* __restrict__ send,
                                  int kpz, int nx, int ny, long long ldm,
                                  const int* __restrict__ ys, int parts) {
  const long long total = (long long)kpz * nx * ny;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e % ny);
    const long long row = e / ny;  // l * nx + n
    long long base;
    int kp;
    const int q = owner_of(ys, parts, m, base, kp, (long long)kpz * nx);
    send[base + row * kp + (m - ys[q])] = modes[row * ldm + m];
  }
}

__global__ void unpack_modes_kernel(const double* __restrict__ recv, double* __restrict__ modes,
                                    int kpz, int nx, int ny, long long ldm,
                                    const int* __restrict__ ys, int parts) {
  const long long total = (long long)kpz * nx * ny;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e % ny);
    const long long row = e / ny;
    long long base;
    int kp;
    const int q = owner_of(ys, parts, m, base, kp, (long long)kpz * nx);
    modes[row * ldm + m] = recv[base + row * kp + (m - ys[q])];
  }
}

extern "C" int hfb_modes_ld(const hfb_plan* p) { return p ? (int)modes_ld(p) : 0; }

extern "C" int hfb_forward_modes(hfb_plan* p, const double* src, double* modes, void* work,
                                 void* stream) {
  const NvtxRange nvtx_("hfb_forward_modes");
  if (!p || !src || !modes || !work) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  return forward_modes(p, src, modes, (double*)work, (cudaStream_t)stream);
}

// kp of the uniform exchange geometry (every part's y-range rounded up to even is
// the same kp and parts * kp = n_y + 1, whole 128-byte segments), else 0
static int uniform_kp(const hfb_plan* p, const int* ys, int parts) {
  if (!ys || parts < 1 || ys[0] != 0 || ys[parts] != p->ny) return 0;
  const int kp = (p->ny + 1) / parts;
  if (kp * parts != p->ny + 1 || kp % 16) return 0;
  for (int q = 0; q < parts; ++q)
    if (ys[q] != q * kp) return 0;
  return kp;
}

extern "C" int hfb_forward_blocks(hfb_plan* p, const double* src, double* send, void* work,
                                  const int* ys, int parts, void* stream) {
  const NvtxRange nvtx_("hfb_forward_blocks");
  if (!p || !src || !send || !work) return HFB_ERR_ARGUMENT;
  const int kp = uniform_kp(p, ys, parts);
  if (!kp) return HFB_ERR_PARTITION;
  HFB_CUDA(cudaSetDevice(p->device));
  return forward_modes(p, src, send, (double*)work, (cudaStream_t)stream, parts, kp);
}

extern "C" int hfb_inverse_blocks(hfb_plan* p, const double* back, double* modes, double* out,
                                  const int* ys, int parts, void* stream) {
  const NvtxRange nvtx_("hfb_inverse_blocks");
  if (!p || !back || !modes || !out) return HFB_ERR_ARGUMENT;
  const int kp = uniform_kp(p, ys, parts);
  if (!kp) return HFB_ERR_PARTITION;
  HFB_CUDA(cudaSetDevice(p->device));
  return inverse_modes_blocks(p, back, modes, out, parts, kp, (cudaStream_t)stream);
}

extern "C" int hfb_inverse_modes(hfb_plan* p, double* modes, double* out, void* stream) {
  const NvtxRange nvtx_("hfb_inverse_modes");
  if (!p || !modes || !out) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  return inverse_modes(p, modes, out, (cudaStream_t)stream);
}

extern "C" int hfb_solve_modes(hfb_plan* p, double* data, int ld, int m_count, int m_offset,
                               void* cp_work, void* stream) {
  const NvtxRange nvtx_("hfb_solve_modes");
  if (!p || !data || !cp_work || ld < m_count || (ld & 1)) return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;
  if (m_count < 0 || m_offset < 0 || m_offset + m_count > p->ny) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas_tma_cols(p, data, (double*)cp_work, ld, (long long)ld * p->nx, m_count,
                                m_offset, (cudaStream_t)stream);
}

extern "C" int hfb_solve_modes_perm(hfb_plan* p, double* data, int ld, int m_count,
                                    int m_offset, const int* level_plane, void* cp_work,
                                    void* stream) {
  if (!p || !data || !cp_work || !level_plane || ld < m_count || (ld & 1))
    return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;
  if (m_count < 0 || m_offset < 0 || m_offset + m_count > p->ny) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (p->lvlmap_cap < p->nz) {
    if (p->lvlmap) cudaFree(p->lvlmap);
    p->lvlmap = nullptr;
    HFB_CUDA(cudaMalloc(&p->lvlmap, sizeof(int) * p->nz));
    p->lvlmap_cap = p->nz;
  }
  HFB_CUDA(cudaMemcpyAsync(p->lvlmap, level_plane, sizeof(int) * p->nz, cudaMemcpyHostToDevice,
                           st));
  return launch_thomas_tma_cols(p, data, (double*)cp_work, ld, (long long)ld * p->nx, m_count,
                                m_offset, st, 0, 0, -1, 0, p->lvlmap);
}

extern "C" int hfb_pack_modes(hfb_plan* p, const double* modes, double* send, const int* ys,
                              int parts, void* stream) {
  if (!p || !modes || !send || !ys || parts < 1) return HFB_ERR_ARGUMENT;
  if (ys[0] != 0 || ys[parts] != p->ny) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  int rc = upload_ystarts(p, ys, parts, (cudaStream_t)stream);
  if (rc) return rc;
  const long long n = (long long)p->nz * p->nx * p->ny;
  if (n == 0) return HFB_OK;
  pack_modes_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      modes, send, p->nz, p->nx, p->ny, modes_ld(p), p->ystarts, parts);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_unpack_modes(hfb_plan* p, const double* recv, double* modes, const int* ys,
                                int parts, void* stream) {
  if (!p || !modes || !recv || !ys || parts < 1) return HFB_ERR_ARGUMENT;
  if (ys[0] != 0 || ys[parts] != p->ny) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  int rc = upload_ystarts(p, ys, parts, (cudaStream_t)stream);
  if (rc) return rc;
  const long long n = (long long)p->nz * p->nx * p->ny;
  if (n == 0) return HFB_OK;
  unpack_modes_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      recv, modes, p->nz, p->nx, p->ny, modes_ld(p), p->ystarts, parts);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_rhs_sixth_z(hfb_plan* p, const double* const* fields_re,
                               const double* const* fields_im, const double* k2_re,
                               const double* k2_im, const double* k2z_re, const double* k2z_im,
                               double h2, double* F_re, double* F_im, void* stream) {
  if (!p || !fields_re || !fields_im || !k2_re || !k2_im || !k2z_re || !k2z_im || !F_re ||
      !F_im)
    return HFB_ERR_ARGUMENT;
  Fields7 fr, fi;
  for (int k = 0; k < 7; ++k) {
    if (!fields_re[k] || !fields_im[k]) return HFB_ERR_ARGUMENT;
    fr.p[k] = fields_re[k];
    fi.p[k] = fields_im[k];
  }
  HFB_CUDA(cudaSetDevice(p->device));
  const long long plane = (long long)p->nx * p->ny, n = plane * p->nz;
  rhs_sixth_z_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      fr, fi, k2_re, k2_im, k2z_re, k2z_im, h2, plane, n, F_re, F_im);
  HFB_LAUNCHED();
  return HFB_OK;
}

extern "C" int hfb_rhs_convdiff_z(hfb_plan* p, const double* const* fields_re,
                                  const double* const* fields_im, double hx2, double hy2,
                                  double hz2, double gamma_re, double gamma_im, double* F_re,
                                  double* F_im, void* stream) {
  if (!p || !fields_re || !fields_im || !F_re || !F_im) return HFB_ERR_ARGUMENT;
  Fields7 fr = {}, fi = {};
  for (int k = 0; k < 5; ++k) {
    if (!fields_re[k] || !fields_im[k]) return HFB_ERR_ARGUMENT;
    fr.p[k] = fields_re[k];
    fi.p[k] = fields_im[k];
  }
  HFB_CUDA(cudaSetDevice(p->device));
  const long long n = (long long)p->nx * p->ny * p->nz;
  rhs_convdiff_z_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      fr, fi, hx2, hy2, hz2, gamma_re, gamma_im, n, F_re, F_im);
  HFB_LAUNCHED();
  return HFB_OK;
}
