// Complex-coefficient z-solve (complex k(z)).
//
// Same streaming structure as thomas_tma.cu — a CTA owns BM = 256 consecutive
// modes (n fixed, m0..m0+255), levels stream through a 3-stage shared-memory
// ring in chunks of K = 8 by 1D bulk copies, cp is checkpointed once per chunk
// and recomputed bitwise in the back substitution — with the data held as two
// real volumes (real and imaginary parts, same padded (l, n, m) layout) and
// complex eigenvalues lambda = 4a cx cy + 2b cx + 2c cy + d from complex
// per-level weights (stencil.py:226-234 with complex a..d; tridiag.py:126-167
// in complex arithmetic). A pivot fails when |den| < PIVOT_RTOL * scale, as
// the reference's abs() of a complex denominator (tridiag.py:136-151).
#include "hfb_internal.cuh"
#include "tma.cuh"

namespace hfb {

namespace {
constexpr int BM = 256;
constexpr int K = kThomasChunk;
constexpr int S = 3;

struct TmaZArgs {
  int xsparse;          // x' stored once per chunk, recomputed (thomas_tma.cu, key 23)
  double* wr;           // real parts (l, n, m): x' / W in place
  double* wi;           // imaginary parts, same layout
  double* cpk;          // checkpoints: planes 2q (re) and 2q+1 (im) for chunk q
  const double* coefr;  // [l][k][(4a, 2b, 2c, d)] real parts
  const double* coefi;  // imaginary parts
  const double* cx;
  const double* cy;
  int nz, nrows, ncols, nbpr;
  long long ld, ps;
  double thr2;  // (PIVOT_RTOL * scale)^2
  unsigned long long* err;
  int nx, ny_total;
};

struct cz {
  double r, i;
};

__device__ __forceinline__ double eig_z(const double* co, double cx, double cy, double cxy) {
  return fma(co[0], cxy, fma(co[1], cx, fma(co[2], cy, co[3])));
}
__device__ __forceinline__ cz zmul(cz a, cz b) {
  return {fma(a.r, b.r, -a.i * b.i), fma(a.r, b.i, a.i * b.r)};
}
// a - b * c
__device__ __forceinline__ cz zfms(cz a, cz b, cz c) {
  return {fma(-b.r, c.r, fma(b.i, c.i, a.r)), fma(-b.r, c.i, fma(-b.i, c.r, a.i))};
}
__device__ __forceinline__ cz zrcp(cz d, double& n2) {
  n2 = fma(d.r, d.r, d.i * d.i);
  const double inv = rcp_fast(n2);  // bitwise 1.0 / n2 for normal n2
  return {d.r * inv, -d.i * inv};
}
}  // namespace

__global__ void __launch_bounds__(BM) thomas_tma_z_kernel(TmaZArgs a) {
  extern __shared__ __align__(16) double dyn[];
  // stage s: [2][K][BM] data (re, im), then [2][K * 12] weights (re, im)
  double(*sdat)[2][K][BM] = reinterpret_cast<double(*)[2][K][BM]>(dyn);
  double(*scoef)[2][K * 12] = reinterpret_cast<double(*)[2][K * 12]>(dyn + S * 2 * K * BM);
  __shared__ uint64_t bar[S];
  const int tid = threadIdx.x;
  const int nchunk = (a.nz + K - 1) / K;
  const int ntask = 2 * nchunk;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase = 0;

  for (long long blk = blockIdx.x; blk < (long long)a.nrows * a.nbpr; blk += gridDim.x) {
    const int n = (int)(blk / a.nbpr);
    const int m0 = (int)(blk % a.nbpr) * BM;
    const int cols = min(BM, a.ncols - m0);
    const uint32_t rowbytes = (uint32_t)(((cols + 1) & ~1) * 8);
    const long long boff = (long long)n * a.ld + m0;
    auto chunk_of = [&](int task) { return task < nchunk ? task : ntask - 1 - task; };
    auto issue = [&](int task, int s) {
      const int c = chunk_of(task);
      const int l0 = c * K, nl = min(K, a.nz - l0);
      mbar_arrive_expect_tx(&bar[s], 2 * nl * rowbytes + (uint32_t)(2 * nl * 12 * 8));
      for (int i = 0; i < nl; ++i) {
        const long long off = boff + (long long)(l0 + i) * a.ps;
        bulk_g2s(&sdat[s][0][i][0], a.wr + off, rowbytes, &bar[s]);
        bulk_g2s(&sdat[s][1][i][0], a.wi + off, rowbytes, &bar[s]);
      }
      bulk_g2s(&scoef[s][0][0], a.coefr + (long long)l0 * 12, (uint32_t)(nl * 12 * 8), &bar[s]);
      bulk_g2s(&scoef[s][1][0], a.coefi + (long long)l0 * 12, (uint32_t)(nl * 12 * 8), &bar[s]);
    };
    const bool live = tid < cols;
    const int m = m0 + tid;
    const double cxv = __ldg(a.cx + n);
    const double cyv = live ? __ldg(a.cy + m) : 0.0;
    const double cxy = cxv * cyv;
    double* ck = a.cpk + boff + tid;  // chunk q: re at plane 2q, im at 2q + 1
    auto stage_of = [&](int task) { return task < nchunk ? task % S : (task - 1) % S; };
    auto needs_load = [&](int task) { return task != nchunk; };
    auto lam = [&](int s, int i, int k) -> cz {
      return {eig_z(&scoef[s][0][i * 12 + 4 * k], cxv, cyv, cxy),
              eig_z(&scoef[s][1][i * 12 + 4 * k], cxv, cyv, cxy)};
    };
    if (tid == 0) {
      issue(0, stage_of(0));
      if (ntask > 1 && needs_load(1)) issue(1, stage_of(1));
    }
    cz c = {0.0, 0.0}, x = {0.0, 0.0}, cknext = {0.0, 0.0};
    for (int task = 0; task < ntask; ++task) {
      const int s = stage_of(task);
      if (tid == 0 && task + 2 < ntask && needs_load(task + 2)) {
        if (task + 2 > nchunk) bulk_wait<0>(); else bulk_wait_read<0>();
        fence_proxy_async_smem();
        issue(task + 2, stage_of(task + 2));
      }
      if (needs_load(task)) {
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
      }
      const int cidx = chunk_of(task);
      const int l0 = cidx * K, nl = min(K, a.nz - l0);
      if (task < nchunk) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i < nl) {
            const int l = l0 + i;
            const cz lo = lam(s, i, 0), di = lam(s, i, 1), up = lam(s, i, 2);
            const cz den = (l == 0) ? di : zfms(di, lo, c);
            double n2;
            const cz rr = zrcp(den, n2);
            if (live && !(n2 >= a.thr2)) {
              const unsigned long long key =
                  ((unsigned long long)l * (unsigned long long)a.ny_total + (unsigned long long)m) *
                      (unsigned long long)a.nx +
                  (unsigned long long)n;
              atomicMin(a.err, key);
            }
            const cz f = {sdat[s][0][i][tid], sdat[s][1][i][tid]};
            x = zmul((l == 0) ? f : zfms(f, lo, x), rr);
            if (!a.xsparse || i == 0 || task == nchunk - 1) {
              sdat[s][0][i][tid] = x.r;
              sdat[s][1][i][tid] = x.i;
            }
            if (l < a.nz - 1) {
              c = zmul(up, rr);
              if (i == K - 1 && live) {
                ck[(long long)(2 * cidx) * a.ps] = c.r;
                ck[(long long)(2 * cidx + 1) * a.ps] = c.i;
              }
            }
          }
        }
        if (live && task == nchunk - 1 && nchunk > 1)
          cknext = {ck[(long long)(2 * (nchunk - 2)) * a.ps],
                    ck[(long long)(2 * (nchunk - 2) + 1) * a.ps]};
      } else {
        cz cprev = cknext;
        if (cidx >= 2 && live)
          cknext = {ck[(long long)(2 * (cidx - 2)) * a.ps],
                    ck[(long long)(2 * (cidx - 2) + 1) * a.ps]};
        cz cb[K];
        // sparse x': recompute the chunk's rows from its stored first row with the
        // forward's expressions (every chunk but the on-chip last one)
        const bool rec = a.xsparse && task != nchunk;
        cz xr = rec ? cz{sdat[s][0][0][tid], sdat[s][1][0][tid]} : cz{0.0, 0.0};
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int l = l0 + i;
          if (i < nl && l < a.nz - 1) {
            const cz di = lam(s, i, 1);
            const cz lo = lam(s, i, 0);
            const cz dl = (l == 0) ? di : zfms(di, lo, cprev);
            double n2;
            const cz rr = zrcp(dl, n2);
            if (rec && i > 0) {
              xr = zmul(zfms({sdat[s][0][i][tid], sdat[s][1][i][tid]}, lo, xr), rr);
              sdat[s][0][i][tid] = xr.r;
              sdat[s][1][i][tid] = xr.i;
            }
            cprev = zmul(lam(s, i, 2), rr);
            cb[i] = cprev;
          }
        }
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
          const int l = l0 + i;
          if (i < nl && l < a.nz - 1) {
            x = zfms({sdat[s][0][i][tid], sdat[s][1][i][tid]}, cb[i], x);
            sdat[s][0][i][tid] = x.r;
            sdat[s][1][i][tid] = x.i;
          }
        }
      }
      __syncthreads();
      if (tid == 0 && task != nchunk - 1) {
        fence_proxy_async_smem();
        const int nst = (a.xsparse && task < nchunk) ? 1 : nl;  // sparse x': level l0 only
        for (int i = 0; i < nst; ++i) {
          const long long off = boff + (long long)(l0 + i) * a.ps;
          bulk_s2g(a.wr + off, &sdat[s][0][i][0], rowbytes);
          bulk_s2g(a.wi + off, &sdat[s][1][i][0], rowbytes);
        }
        bulk_commit();
      }
    }
    if (tid == 0) bulk_wait<0>();
    __syncthreads();
  }
}

int launch_thomas_tma_z(hfb_plan* p, double* re, double* im, double* cpk, long long ld,
                        long long ps, cudaStream_t st) {
  if (p->nz < 1) return HFB_OK;
  if (!p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  TmaZArgs a;
  a.xsparse = tuning(23);
  a.wr = re;
  a.wi = im;
  a.cpk = cpk;
  a.coefr = p->coef;
  a.coefi = p->coef_i;
  a.cx = p->cx;
  a.cy = p->cy;
  a.nz = p->nz;
  a.nrows = p->nx;
  a.ncols = p->ny;
  a.nbpr = (p->ny + BM - 1) / BM;
  a.ld = ld;
  a.ps = ps;
  a.thr2 = p->thr * p->thr;
  a.err = p->err;
  a.nx = p->nx;
  a.ny_total = p->ny;
  const size_t sm = sizeof(double) * (size_t)S * 2 * (K * BM + K * 12);
  HFB_CUDA(cudaFuncSetAttribute(thomas_tma_z_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, thomas_tma_z_kernel, BM, sm));
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nrows * a.nbpr;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  thomas_tma_z_kernel<<<(unsigned)blocks, BM, sm, st>>>(a);
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb

// ----------------------------------------------------------------------
// Complex z-solve on a natural-layout slab (l, m, n): thread per mode, rows
// m_off + r (y-modes) of the full grid, columns n (x-modes); cp (complex) is
// kept whole in a workspace of two slab volumes. Used by the generic-size
// path of hfb_solve_z and by hfb_solve_slab_z (the partitioned mode).
namespace hfb {
namespace {
struct SlabZArgs {
  double *wr, *wi, *cr, *ci;
  const double *coefr, *coefi, *cx, *cy;
  int nz, mloc, nx, ny_total, m_off;
  long long ps;  // plane stride = mloc * nx
  double thr2;
  unsigned long long* err;
};
}  // namespace

__global__ void __launch_bounds__(256) thomas_slab_z_kernel(SlabZArgs a) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)a.mloc * a.nx) return;
  const int r = (int)(t / a.nx), n = (int)(t - (long long)r * a.nx);
  const int m = a.m_off + r;
  const double cxv = __ldg(a.cx + n), cyv = __ldg(a.cy + m), cxy = cxv * cyv;
  auto lam = [&](int l, int k) -> cz {
    return {eig_z(a.coefr + (long long)l * 12 + 4 * k, cxv, cyv, cxy),
            eig_z(a.coefi + (long long)l * 12 + 4 * k, cxv, cyv, cxy)};
  };
  cz c = {0.0, 0.0}, x = {0.0, 0.0};
  for (int l = 0; l < a.nz; ++l) {
    const long long e = (long long)l * a.ps + t;
    const cz lo = lam(l, 0), di = lam(l, 1);
    const cz den = (l == 0) ? di : zfms(di, lo, c);
    double n2;
    const cz rr = zrcp(den, n2);
    if (!(n2 >= a.thr2)) {
      const unsigned long long key =
          ((unsigned long long)l * (unsigned long long)a.ny_total + (unsigned long long)m) *
              (unsigned long long)a.nx +
          (unsigned long long)n;
      atomicMin(a.err, key);
    }
    const cz f = {a.wr[e], a.wi[e]};
    x = zmul((l == 0) ? f : zfms(f, lo, x), rr);
    a.wr[e] = x.r;
    a.wi[e] = x.i;
    if (l < a.nz - 1) {
      c = zmul(lam(l, 2), rr);
      a.cr[e] = c.r;
      a.ci[e] = c.i;
    }
  }
  for (int l = a.nz - 2; l >= 0; --l) {
    const long long e = (long long)l * a.ps + t;
    x = zfms({a.wr[e], a.wi[e]}, {a.cr[e], a.ci[e]}, x);
    a.wr[e] = x.r;
    a.wi[e] = x.i;
  }
}

int launch_thomas_slab_z(hfb_plan* p, double* re, double* im, int mloc, int m_off, double* cpw,
                         cudaStream_t st) {
  if (p->nz < 1 || mloc < 1) return HFB_OK;
  if (!p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  SlabZArgs a;
  a.wr = re;
  a.wi = im;
  a.ps = (long long)mloc * p->nx;
  a.cr = cpw;
  a.ci = cpw + a.ps * p->nz;
  a.coefr = p->coef;
  a.coefi = p->coef_i;
  a.cx = p->cx;
  a.cy = p->cy;
  a.nz = p->nz;
  a.mloc = mloc;
  a.nx = p->nx;
  a.ny_total = p->ny;
  a.m_off = m_off;
  a.thr2 = p->thr * p->thr;
  a.err = p->err;
  const long long modes = (long long)mloc * p->nx;
  thomas_slab_z_kernel<<<(unsigned)((modes + 255) / 256), 256, 0, st>>>(a);
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb
