// Batched orthonormal DST-I along x (contiguous lines) and along y (strided
// columns) — kernels (b)/(d) of the north star, replacing
// spectral.dst_lines / transform_stack / transform_lines_x/y
// (reference spectral.py:54-111).
//
// Power-of-two N+1: one complex Stockham FFT per pair of real lines, in
// shared memory (hfb_internal.cuh). Other N: dense DST-I matrix product
// (fp64 GEMM, S symmetric), out of place through a temporary.
#include <algorithm>

#include "hfb_internal.cuh"

namespace hfb {

// Threads per transform group for length M.
static inline int group_threads(int M) { return M >= 8 ? M / 8 : 1; }

struct LineSet {
  // rows y0 + 2k, y0 + 2k + 1 of one plane form pair k; pairs never straddle
  // planes, so a plane range never changes which rows share an FFT (results
  // are bitwise independent of how the planes are split)
  int z0, y0, nrow, ppp;  // ppp = pairs per plane = ceil(nrow / 2)
  long long npairs;
  long long ld, ps;       // row and plane strides (elements)
};

// x-pass: CTA = B groups of G threads; group f transforms one row pair as one
// complex FFT (real part = even row, imaginary part = odd row).
__global__ void __launch_bounds__(512) dst_x_fft_kernel(const double* __restrict__ src,
                                                         double* __restrict__ dst, LineSet s,
                                                         int N, FftCtx c, int B) {
  extern __shared__ double2 smem[];
  const int f = threadIdx.x / c.G, g = threadIdx.x % c.G;
  double2* buf = smem + f * (c.M + 1);
  double2* wsum = smem + B * (c.M + 1);
  const long long pair = (long long)blockIdx.x * B + f;
  const bool live = pair < s.npairs;
  const long long pl = live ? s.z0 + pair / s.ppp : 0;
  const int r0 = live ? 2 * (int)(pair % s.ppp) : 0;
  const bool v0 = live, v1 = live && r0 + 1 < s.nrow;
  const long long o0 = pl * s.ps + (long long)(s.y0 + r0) * s.ld;
  const long long o1 = o0 + s.ld;
  for (int j = g; j < N; j += c.G) {
    const double x = v0 ? src[o0 + j] : 0.0;
    const double y = v1 ? src[o1 + j] : 0.0;
    buf[j + 1] = make_double2(x, y);
  }
  __syncthreads();
  dst_core(buf, c, g, wsum);
  for (int p = g; p < N; p += c.G) {
    const double2 o = buf[p];
    if (v0) dst[o0 + p] = o.x;
    if (v1) dst[o1 + p] = o.y;
  }
}

// y-pass: CTA = one plane x a tile of 2B columns; group f transforms the
// column pair (c0 + 2f, c0 + 2f + 1) as one complex FFT. Loads and stores
// are row-major over the tile (coalesced), staged through shared memory.
__global__ void __launch_bounds__(512) dst_y_fft_kernel(const double* __restrict__ src,
                                                         double* __restrict__ dst, int z0,
                                                         int x0, int x1, long long ld,
                                                         long long ps, int N, FftCtx c, int B,
                                                         int nplanes) {
  extern __shared__ double2 smem[];
  const int f = threadIdx.x / c.G, g = threadIdx.x % c.G;
  const int W = 2 * B;
  double2* wsum = smem + B * (c.M + 1);
  double* sb = reinterpret_cast<double*>(smem);
  const int col0 = x0 + blockIdx.x * W;
  const int ncols = min(W, x1 - col0);
  const int total = N * W;
  // planes z0 + blockIdx.y + k gridDim.y (gridDim.y <= 65535)
  for (long long plane = z0 + blockIdx.y; plane < z0 + nplanes; plane += gridDim.y) {
    const double* P = src + plane * ps + col0;
    double* Q = dst + plane * ps + col0;
    __syncthreads();  // the previous plane's stores have read shared memory
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int row = e / W, col = e - row * W;
      const double v = col < ncols ? P[row * ld + col] : 0.0;
      sb[2 * ((col >> 1) * (c.M + 1) + row + 1) + (col & 1)] = v;
    }
    __syncthreads();
    dst_core(smem + f * (c.M + 1), c, g, wsum);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int row = e / W, col = e - row * W;
      if (col < ncols) Q[row * ld + col] = sb[2 * ((col >> 1) * (c.M + 1) + row) + (col & 1)];
    }
  }
}

// ------------------------------------------------------------ dense path
// C[b] = A[b] * B[b], row-major, Mr x Kd times Kd x Nc; 64x64 tiles, 256
// threads, 4x4 outputs per thread.
__global__ void __launch_bounds__(256) dgemm_batched_kernel(
    int Mr, int Nc, int Kd, const double* __restrict__ A, long long lda, long long sA,
    const double* __restrict__ Bm, long long ldb, long long sB, double* __restrict__ C,
    long long ldc, long long sC) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int b = blockIdx.z;
  A += b * sA;
  Bm += b * sB;
  C += b * sC;
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < Kd; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e % 16, r = e / 16;  // A tile: 64 rows x 16 k
      const int gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < Mr && gk < Kd) ? A[gr * lda + gk] : 0.0;
      const int cc = e % 64, kb = e / 64;  // B tile: 16 k x 64 cols
      const int gk2 = k0 + kb, gc = col0 + cc;
      Bs[kb][cc] = (gk2 < Kd && gc < Nc) ? Bm[gk2 * ldb + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tc + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = row0 + tr + 16 * i, cc = col0 + tc + 16 * j;
      if (r < Mr && cc < Nc) C[r * ldc + cc] = acc[i][j];
    }
}

// The same product on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): 64x64
// CTA tiles, 4 warps of 32x32 (4 x 4 m8n8 accumulators each), k in blocks of 16
// staged through shared memory as in dgemm_batched_kernel. Fragments (PTX
// m8n8k4 .f64): A[r = lane/4][k = lane%4], B[k = lane%4][c = lane/4],
// C[r = lane/4][c = 2 (lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) dmma_batched_kernel(
    int Mr, int Nc, int Kd, const double* __restrict__ A, long long lda, long long sA,
    const double* __restrict__ Bm, long long ldb, long long sB, double* __restrict__ C,
    long long ldc, long long sC) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int b = blockIdx.z;
  A += b * sA;
  Bm += b * sB;
  C += b * sC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
  const int row0 = blockIdx.y * 64, col0 = blockIdx.x * 64;
  const int fr = lane >> 2, fk = lane & 3;
  double acc[4][4][2] = {};
  for (int k0 = 0; k0 < Kd; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 128) {
      const int kk = e % 16, r = e / 16;  // A tile: 64 rows x 16 k
      const int gr = row0 + r, gk = k0 + kk;
      As[kk][r] = (gr < Mr && gk < Kd) ? A[gr * lda + gk] : 0.0;
      const int cc = e % 64, kb = e / 64;  // B tile: 16 k x 64 cols
      const int gk2 = k0 + kb, gc = col0 + cc;
      Bs[kb][cc] = (gk2 < Kd && gc < Nc) ? Bm[gk2 * ldb + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < 16; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[ks + fk][wr + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[ks + fk][wc + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = row0 + wr + 8 * i + fr, cc = col0 + wc + 8 * j + 2 * fk + h;
        if (r < Mr && cc < Nc) C[r * ldc + cc] = acc[i][j][h];
      }
}

// Small-N 2D DST-I of whole planes on the FP64 tensor cores (the reference's
// per-plane dst2d, spectral.py:54-72, written as the dense product its own
// test checks against: dst2d_reference / oracle.dense_sine_matrix,
// spectral.py:66-72, oracle.py:106-109): Y = S_y X S_x
// (S symmetric, orthonormal scale included) with X, the intermediate T = X S_x,
// and both S in shared memory, zero-padded to NP x NP (NP = 32 or 64). One
// plane per CTA iteration, persistent over planes: 16 B/point of HBM traffic
// for the whole 2D transform (one read, one write of a contiguous plane) and
// 4 NP flops per point on DMMA (mma.sync.m8n8k4.f64). Warp w owns output rows
// [8w, 8w + 8) of each product, all NP/8 column tiles.
// Layouts: natural planes (row j = y position, ld = row stride, x fastest) or
// mode rows (row n = x mode, y modes m fastest — the one-call solve's and the
// partitioned path's (l, n, m) layout). tin: the input is mode rows (read
// transposed, W[n][m] -> X[m][n]); tout: write Y[m][n] as mode rows (n, m).
struct D2Layout {
  long long ld_in, ps_in, ld_out, ps_out;
  int tin, tout;
};

template <int NP>
__global__ void __launch_bounds__(4 * NP) dmma_dst2d_kernel(const double* src, double* dst,
                                                            int z0, int nz, int nx, int ny,
                                                            const double* __restrict__ Sx,
                                                            const double* __restrict__ Sy,
                                                            D2Layout lay) {
  constexpr int LD = NP + 1, NT = NP / 8;
  extern __shared__ double sm2[];
  double* xs = sm2;              // X, then Y
  double* ts = xs + NP * LD;     // T = X S_x
  double* sx = ts + NP * LD;
  double* sy = sx + NP * LD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fr = lane >> 2, fk = lane & 3;
  const int nth = blockDim.x;
  for (int e = threadIdx.x; e < NP * NP; e += nth) {
    const int r = e / NP, c = e % NP;
    sx[r * LD + c] = (r < nx && c < nx) ? __ldg(Sx + r * nx + c) : 0.0;
    sy[r * LD + c] = (r < ny && c < ny) ? __ldg(Sy + r * ny + c) : 0.0;
  }
  for (int pl = blockIdx.x; pl < nz; pl += gridDim.x) {
    const double* X = src + (long long)(z0 + pl) * lay.ps_in;
    __syncthreads();  // the previous plane's Y has been stored
    if (!lay.tin) {
      for (int e = threadIdx.x; e < NP * NP; e += nth) {
        const int r = e / NP, c = e % NP;
        xs[r * LD + c] = (r < ny && c < nx) ? X[r * lay.ld_in + c] : 0.0;
      }
    } else {  // mode rows: element (n, m) at X[n ld + m] -> xs[m][n]
      for (int e = threadIdx.x; e < NP * NP; e += nth) {
        const int n = e / NP, m = e % NP;
        xs[m * LD + n] = (n < nx && m < ny) ? X[n * lay.ld_in + m] : 0.0;
      }
    }
    __syncthreads();
    // T = X S_x (rows of X: y positions j, columns: x modes n)
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NP; ks += 4) {
      const double a = xs[(8 * warp + fr) * LD + ks + fk];
#pragma unroll
      for (int j = 0; j < NT; ++j)
        dmma884(acc[j][0], acc[j][1], a, sx[(ks + fk) * LD + 8 * j + fr]);
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      ts[(8 * warp + fr) * LD + 8 * j + 2 * fk] = acc[j][0];
      ts[(8 * warp + fr) * LD + 8 * j + 2 * fk + 1] = acc[j][1];
    }
    __syncthreads();
    // Y = S_y T (rows: y modes m)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NP; ks += 4) {
      const double a = sy[(8 * warp + fr) * LD + ks + fk];
#pragma unroll
      for (int j = 0; j < NT; ++j)
        dmma884(acc[j][0], acc[j][1], a, ts[(ks + fk) * LD + 8 * j + fr]);
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      xs[(8 * warp + fr) * LD + 8 * j + 2 * fk] = acc[j][0];
      xs[(8 * warp + fr) * LD + 8 * j + 2 * fk + 1] = acc[j][1];
    }
    __syncthreads();
    double* Y = dst + (long long)(z0 + pl) * lay.ps_out;
    if (!lay.tout) {
      for (int e = threadIdx.x; e < nx * ny; e += nth) {
        const int r = e / nx, c = e - r * nx;
        Y[r * lay.ld_out + c] = xs[r * LD + c];
      }
    } else {  // mode rows (n, m): Y[n ld + m] = xs[m][n]
      for (int e = threadIdx.x; e < nx * ny; e += nth) {
        const int n = e / ny, m = e - n * ny;
        Y[n * lay.ld_out + m] = xs[m * LD + n];
      }
    }
  }
}

// Where the whole-plane DMMA transform is used (tools/dense_bench.py on a B200,
// ~32 MB stacks, 2D transform): N = 31 0.43 ms against 0.74 for the FFT engine;
// N = 15 1.56 vs 1.46 (FFT); N = 63 (64-padded tiles) 0.82 vs 0.53 (FFT); N = 40
// 1.79 vs 1.45 for the two-pass dense GEMM. So: lines of at most 32 (tuning key
// 18, default 32; 0 = never), and at least 16 where the FFT engine applies.
static int dmma2d_np(const hfb_plan* p) {
  const int lim = tuning(18);
  const int n = std::max(p->nx, p->ny);
  if (lim <= 0 || n > lim || n > 64) return 0;
  if (n < 16 && dst16_ok(p->nx + 1) && dst16_ok(p->ny + 1)) return 0;
  return n <= 32 ? 32 : 64;
}

static int launch_dmma2d(hfb_plan* p, const double* src, double* dst, int z0, int z1,
                         cudaStream_t st, const D2Layout* layout = nullptr) {
  const int np = dmma2d_np(p);
  int rc = ensure_dense(p);
  if (rc) return rc;
  const size_t sm = sizeof(double) * 4 * (size_t)np * (np + 1);
  auto kern = np == 32 ? dmma_dst2d_kernel<32> : dmma_dst2d_kernel<64>;
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 4 * np, sm));
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nz = z1 - z0;
  const int blocks = std::max(1, std::min(nz, sms * std::max(per_sm, 1)));
  D2Layout nat = {p->nx, (long long)p->nx * p->ny, p->nx, (long long)p->nx * p->ny, 0, 0};
  kern<<<blocks, 4 * np, sm, st>>>(src, dst, z0, nz, p->nx, p->ny, p->dense_x, p->dense_y,
                                   layout ? *layout : nat);
  HFB_LAUNCHED();
  return HFB_OK;
}

// batched dense product: the DMMA kernel (tuning key 16 = 1, default) or the
// CUDA-core one (0)
static int launch_dense_gemm(int Mr, int Nc, int Kd, const double* A, long long lda, long long sA,
                             const double* Bm, long long ldb, long long sB, double* C,
                             long long ldc, long long sC, int batch, cudaStream_t st) {
  // gridDim.z is at most 65535: long stacks of small planes go in chunks
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = std::min(batch - b0, 65535);
    dim3 grid((Nc + 63) / 64, (Mr + 63) / 64, nb);
    const double* Ab = A + (long long)b0 * sA;
    const double* Bb = Bm + (long long)b0 * sB;
    double* Cb = C + (long long)b0 * sC;
    if (tuning(16))
      dmma_batched_kernel<<<grid, 128, 0, st>>>(Mr, Nc, Kd, Ab, lda, sA, Bb, ldb, sB, Cb, ldc, sC);
    else
      dgemm_batched_kernel<<<grid, 256, 0, st>>>(Mr, Nc, Kd, Ab, lda, sA, Bb, ldb, sB, Cb, ldc, sC);
    HFB_LAUNCHED();
  }
  return HFB_OK;
}

// Copy a (planes x rows x cols) region between two arrays of equal strides.
__global__ void copy_region_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                   int rows, int cols, long long ld, long long ps,
                                   long long off, int nplanes) {
  for (long long pl = blockIdx.y; pl < nplanes; pl += gridDim.y)
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
         e < (long long)rows * cols; e += (long long)gridDim.x * blockDim.x) {
      const long long r = e / cols, cc = e % cols;
      const long long o = off + pl * ps + r * ld + cc;
      dst[o] = src[o];
    }
}

size_t dense_tmp_elems(const hfb_plan* p, int nplanes) {
  if (p->logMx >= 0 && p->logMy >= 0) return 0;
  return (size_t)nplanes * p->ny * p->nx;
}

static FftCtx make_ctx(int M, int logM, const double2* tw, const double* sn, double scale) {
  FftCtx c;
  c.M = M;
  c.logM = logM;
  c.G = group_threads(M);
  c.tw = tw;
  c.sn = sn;
  c.scale = scale;
  return c;
}

// tuning key 17: lines of length <= key use the dense product even when N + 1
// is a power of two (the FFT / DMMA crossover measurement)
static bool force_dense(const hfb_plan* p) {
  const int lim = tuning(17);
  return lim > 0 && p->nx <= lim && p->ny <= lim;
}

int launch_dst_x(hfb_plan* p, const double* src, double* dst, int z0, int z1, int y0, int y1,
                 double* tmp, cudaStream_t st) {
  const int nz = z1 - z0, nr = y1 - y0;
  if (nz <= 0 || nr <= 0) return HFB_OK;
  const long long ld = p->nx, ps = (long long)p->ny * p->nx;
  const bool dense = force_dense(p);
  if (dense) {
    int rc = ensure_dense(p);
    if (rc) return rc;
  }
  if (!dense && dst16_ok(p->nx + 1)) {
    const long long off = (long long)y0 * ld;
    return launch_dst16(p->tw_x, p->sn_x, p->scale_x, p->nx + 1, src + off,
                        src + (long long)p->nz * ps, dst + off, z0, nz, nr, ld, ps, ld, ps, false,
                        st);
  }
  if (!dense && p->logMx >= 0) {
    const int M = p->nx + 1;
    FftCtx c = make_ctx(M, p->logMx, p->tw_x, p->sn_x, p->scale_x);
    const int B = std::max(1, 256 / c.G);
    const int threads = B * c.G;
    LineSet s;
    s.z0 = z0;
    s.y0 = y0;
    s.nrow = nr;
    s.ppp = (nr + 1) / 2;
    s.npairs = (long long)nz * s.ppp;
    s.ld = ld;
    s.ps = ps;
    const long long blocks = (s.npairs + B - 1) / B;
    const size_t sm = (size_t)(B * (M + 1) + threads / 32 + 1) * sizeof(double2);
    if (sm > 48 * 1024)
      HFB_CUDA(cudaFuncSetAttribute(dst_x_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sm));
    dst_x_fft_kernel<<<(unsigned)blocks, threads, sm, st>>>(src, dst, s, p->nx, c, B);
    HFB_LAUNCHED();
    return HFB_OK;
  }
  // dense: out_l[rows y0..y1) = in_l[rows] * S_x
  if (!tmp) return HFB_ERR_ARGUMENT;
  const double* A = src + (long long)z0 * ps + (long long)y0 * ld;
  double* C = tmp + (long long)z0 * ps + (long long)y0 * ld;
  int rc = launch_dense_gemm(nr, p->nx, p->nx, A, ld, ps, p->dense_x, p->nx, 0, C, ld, ps, nz, st);
  if (rc) return rc;
  dim3 cg(std::max(1, std::min(1024, (nr * p->nx + 255) / 256)), std::min(nz, 65535));
  copy_region_kernel<<<cg, 256, 0, st>>>(tmp, dst, nr, p->nx, ld, ps,
                                         (long long)z0 * ps + (long long)y0 * ld, nz);
  HFB_LAUNCHED();
  return HFB_OK;
}

int launch_dst_y(hfb_plan* p, const double* src, double* dst, int z0, int z1, int x0, int x1,
                 double* tmp, cudaStream_t st) {
  const int nz = z1 - z0, ncol = x1 - x0;
  if (nz <= 0 || ncol <= 0) return HFB_OK;
  const long long ld = p->nx, ps = (long long)p->ny * p->nx;
  const bool dense = force_dense(p);
  if (dense) {
    int rc = ensure_dense(p);
    if (rc) return rc;
  }
  if (!dense && p->logMy >= 0) {
    const int M = p->ny + 1;
    FftCtx c = make_ctx(M, p->logMy, p->tw_y, p->sn_y, p->scale_y);
    int B = std::max(1, 512 / c.G);
    B = std::min(B, 32);
    B = std::min(B, (ncol + 1) / 2 > 0 ? (ncol + 1) / 2 : 1);
    while (B * c.G < 32) ++B;  // keep whole warps
    const int threads = B * c.G;
    const size_t sm = (size_t)(B * (M + 1) + threads / 32 + 1) * sizeof(double2);
    if (sm > 48 * 1024)
      HFB_CUDA(cudaFuncSetAttribute(dst_y_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sm));
    dim3 grid((ncol + 2 * B - 1) / (2 * B), std::min(nz, 65535));
    dst_y_fft_kernel<<<grid, threads, sm, st>>>(src, dst, z0, x0, x1, ld, ps, p->ny, c, B, nz);
    HFB_LAUNCHED();
    return HFB_OK;
  }
  if (!tmp) return HFB_ERR_ARGUMENT;
  const double* Bp = src + (long long)z0 * ps + x0;
  double* C = tmp + (long long)z0 * ps + x0;
  int rc = launch_dense_gemm(p->ny, ncol, p->ny, p->dense_y, p->ny, 0, Bp, ld, ps, C, ld, ps, nz,
                             st);
  if (rc) return rc;
  dim3 cg(std::max(1, std::min(1024, (p->ny * ncol + 255) / 256)), std::min(nz, 65535));
  copy_region_kernel<<<cg, 256, 0, st>>>(tmp, dst, p->ny, ncol, ld, ps, (long long)z0 * ps + x0,
                                         nz);
  HFB_LAUNCHED();
  return HFB_OK;
}

// Transposed scratch line stride for y-lines (even, >= ny).
static long long tran_ld(const hfb_plan* p) { return (p->ny + 1) & ~1LL; }

static bool tran_path(const hfb_plan* p) { return dst16_ok(p->nx + 1) && dst16_ok(p->ny + 1); }

size_t transform_work_elems(const hfb_plan* p, int nplanes) {
  if (tran_path(p)) return (size_t)nplanes * p->nx * tran_ld(p);
  return dense_tmp_elems(p, nplanes);
}

// One-call solve scratch. Every scratch plane holds either (j, n) rows of
// stride ldx or (n, m) rows of stride ldt (both even, so rows are 16-byte
// aligned for the bulk copies and strides are legal for tensor maps); the cp
// checkpoints take one plane per kThomasChunk levels.
//   fast: S1 (x-pass output) + S2 (y-pass output, Thomas, inverse y-pass) + cp
//   lean: S + cp (the forward x-pass writes columns: transposing stores)
static long long x_ld(const hfb_plan* p) { return (p->nx + 1) & ~1LL; }
static long long fused_plane(const hfb_plan* p) {
  return std::max(x_ld(p) * p->ny, tran_ld(p) * p->nx);
}

// Wavefront-fused z-solve (tuning key 21, default on): fast layout, y-lines of
// 511 or 1023 (the fused passes run the M <= 1024 engine with decoupled
// 64-thread groups). Workspace: S1 + S2 + the full cp volume + the W carry
// plane + the level counters.
static bool wave_path(const hfb_plan* p) {
  return tran_path(p) && !p->ws_lean && tuning(21) && (p->ny + 1 == 512 || p->ny + 1 == 1024) &&
         p->nx + 1 <= 4096;
}
static size_t wave_flag_elems(const hfb_plan* p) { return (2 * (size_t)p->nx + 16 + 1) / 2; }

size_t fused_work_elems(const hfb_plan* p) {
  if (!tran_path(p)) return 0;
  if (wave_path(p))
    return (size_t)fused_plane(p) * (3 * (size_t)p->nz + 1) + wave_flag_elems(p);
  const size_t nck = (p->nz + kThomasChunk - 1) / kThomasChunk;
  const size_t arrays = p->ws_lean ? 1 : 2;
  return (size_t)fused_plane(p) * (arrays * p->nz + nck);
}

// The wavefront-fused one-call solve (4 launches):
//   1. x-DST                 F (l, j, i) -> S1 (l, j, n)          [ROW]
//   2. y-DST + forward elim. S1 columns -> S2 x' (l, n, m), CP cp [kYF2]
//   3. back subst. + inv y   S2 x', CP -> S2 (l, n, j)            [kYB, planes descending]
//   4. x-DST                 S2 columns j -> out (l, j, i)        [TLOAD]
// The z-solve's x' round trip of launch 3 of the five-launch schedule is gone:
// x' and cp cross HBM once each way inside the y-passes.
static int solve_wave(hfb_plan* p, const double* rhs, double* out, double* work,
                      cudaStream_t st) {
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), ldx = x_ld(p);
  const long long pst = fused_plane(p);
  double* S1 = work;
  double* S2 = S1 + pst * p->nz;
  double* CP = S2 + pst * p->nz;
  double* WC = CP + pst * p->nz;
  unsigned* flags = reinterpret_cast<unsigned*>(WC + pst);
  HFB_CUDA(cudaMemsetAsync(flags, 0, wave_flag_elems(p) * sizeof(double), st));
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  Dst16Call y = x;
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  int rc;
  const StageMarks mark(p, st);
  mark(0);
  x.mode = 0;  // ROW: F rows -> S1 (l, j, n)
  x.src = rhs;
  x.src_end = rhs + p->nz * ps;
  x.nrow = p->ny;
  x.in_ld = p->nx;
  x.in_ps = ps;
  x.dst = S1;
  x.out_ld = ldx;
  x.out_ps = pst;
  if ((rc = launch_dst16_mode(x, st))) return rc;
  mark(1);
  y.mode = 4;  // kYF2: S1 columns -> S2 x', CP
  y.src = S1;
  y.src_end = S1 + p->nz * pst;
  y.nrow = p->nx;
  y.in_ld = ldx;
  y.in_ps = pst;
  y.dst = S2;
  y.out_ld = ldt;
  y.out_ps = pst;
  y.coef = p->coef;
  y.cx = p->cx;
  y.cy = p->cy;
  y.thr = p->thr;
  y.err = p->err;
  y.cp = CP;
  y.nz_total = p->nz;
  y.flags = flags;
  if ((rc = launch_dst16_mode(y, st))) return rc;
  mark(2);
  mark(3);  // the z-solve rides in launches 2 and 3
  y.mode = 5;  // kYB: S2 x' rows (descending planes) -> S2 (l, n, j)
  y.src = S2;
  y.src_end = S2 + p->nz * pst;
  y.in_ld = ldt;
  y.in_ps = pst;
  y.wc = WC;
  y.flags = flags + p->nx + 8;
  if ((rc = launch_dst16_mode(y, st))) return rc;
  mark(4);
  x.mode = 2;  // TLOAD: S2 columns j -> out (l, j, i)
  x.src = S2;
  x.src_end = S2 + p->nz * pst;
  x.nrow = p->ny;
  x.in_ld = ldt;
  x.in_ps = pst;
  x.dst = out;
  x.out_ld = p->nx;
  x.out_ps = ps;
  if ((rc = launch_dst16_mode(x, st))) return rc;
  mark(5);
  return HFB_OK;
}

// Five launches. Fast layout:
//   1. x-DST   F (l, j, i)    -> S1 (l, j, n)   [ROW: rows in, rows out]
//   2. y-DST   S1 columns n   -> S2 (l, n, m)   [TLOAD: tensor-box columns in, rows out]
//   3. Thomas  per mode (n, m) along l, in place on S2, cp checkpoints
//   4. y-DST   S2 (l, n, .)   -> S2 (l, n, j)   [ROW, in place]
//   5. x-DST   S2 columns j   -> out (l, j, i)  [TLOAD]
// Lean layout replaces 1-2 by an x-pass with transposing stores F -> S (l, n, j)
// and a y-pass in place on S.
int solve_fused(hfb_plan* p, const double* rhs, double* out, double* work, cudaStream_t st) {
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), ldx = x_ld(p);
  const long long pst = fused_plane(p);
  double* S1 = work;
  double* S2 = p->ws_lean ? work : work + pst * p->nz;
  double* CP = S2 + pst * p->nz;
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  Dst16Call y = x;
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  int rc;
  if (wave_path(p) && !dmma2d_np(p)) return solve_wave(p, rhs, out, work, st);
  const StageMarks mark(p, st);
  mark(0);
  if (dmma2d_np(p)) {
    // small N: forward 2D DST of whole planes on DMMA straight into the mode
    // rows, the TMA z-solve, the inverse 2D DST back to natural planes (3
    // launches; the stage slots of the two y-passes stay empty)
    int rc;
    D2Layout fw = {p->nx, ps, ldt, pst, 0, 1}, iv = {ldt, pst, p->nx, ps, 1, 0};
    if ((rc = launch_dmma2d(p, rhs, S2, 0, p->nz, st, &fw))) return rc;
    mark(1);
    mark(2);
    if ((rc = launch_thomas_tma(p, S2, CP, ldt, pst, st, 0))) return rc;
    mark(3);
    mark(4);
    if ((rc = launch_dmma2d(p, S2, out, 0, p->nz, st, &iv))) return rc;
    mark(5);
    return HFB_OK;
  }
  // 1
  x.src = rhs;
  x.src_end = rhs + p->nz * ps;
  x.nrow = p->ny;
  x.in_ld = p->nx;
  x.in_ps = ps;
  if (p->ws_lean) {
    x.mode = 1;  // TRAN: F rows -> S2 (l, n, j)
    x.dst = S2;
    x.out_ld = ldt;
    x.out_ps = pst;
  } else {
    x.mode = 0;  // ROW: F rows -> S1 (l, j, n)
    x.dst = S1;
    x.out_ld = ldx;
    x.out_ps = pst;
  }
  if ((rc = launch_dst16_mode(x, st))) return rc;
  mark(1);
  // 2 (fast layout, fused: the forward Thomas sweep rides in the y-pass)
  const bool fuse = !p->ws_lean && tuning(5);
  y.nrow = p->nx;
  y.dst = S2;
  y.out_ld = ldt;
  y.out_ps = pst;
  if (p->ws_lean) {
    y.mode = 0;  // ROW in place on S2
    y.src = S2;
    y.in_ld = ldt;
  } else {
    y.mode = fuse ? 3 : 2;  // (YF or) TLOAD: S1 columns -> S2 rows
    y.src = S1;
    y.in_ld = ldx;
  }
  y.src_end = y.src + p->nz * pst;
  y.in_ps = pst;
  if (fuse) {
    y.coef = p->coef;
    y.cx = p->cx;
    y.cy = p->cy;
    y.thr = p->thr;
    y.err = p->err;
    y.cp = CP;
    y.nz_total = p->nz;
  }
  // Overlapped schedule (fast layout, unfused): halves of the x-modes n.
  //   st: y-pass n < h | y-pass n >= h (2 CTAs/SM) | . | inverse y n < h (2/SM) | n >= h
  //   B :              | z-solve n < h (1 CTA/SM)  | z-solve n >= h (1/SM)     |
  // The HBM-bound z-solve shares the GPU with the L1-bound y-passes.
  const bool overlap = !p->ws_lean && !fuse && tuning(6) && p->nx >= 64;
  if (overlap) {
    if (!p->ov_stream) {
      HFB_CUDA(cudaStreamCreateWithFlags(&p->ov_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 4; ++i)
        HFB_CUDA(cudaEventCreateWithFlags(&p->ov_ev[i], cudaEventDisableTiming));
    }
    const int h = (p->nx / 2) & ~7;  // a multiple of every line block (4 lines)
    const int cap_dst = tuning(7), cap_th = tuning(8);
    cudaStream_t sb = p->ov_stream;
    Dst16Call ya = y, yb = y;
    ya.line0 = 0;
    ya.line1 = h;
    yb.line0 = h;
    yb.line1 = p->nx;
    yb.max_per_sm = cap_dst;
    if ((rc = launch_dst16_mode(ya, st))) return rc;
    HFB_CUDA(cudaEventRecord(p->ov_ev[0], st));
    if ((rc = launch_dst16_mode(yb, st))) return rc;
    HFB_CUDA(cudaEventRecord(p->ov_ev[1], st));
    mark(2);
    HFB_CUDA(cudaStreamWaitEvent(sb, p->ov_ev[0], 0));
    if ((rc = launch_thomas_tma_cols(p, S2, CP, ldt, pst, p->ny, 0, sb, 0, 0, h, cap_th)))
      return rc;
    HFB_CUDA(cudaEventRecord(p->ov_ev[2], sb));
    HFB_CUDA(cudaStreamWaitEvent(sb, p->ov_ev[1], 0));
    if ((rc = launch_thomas_tma_cols(p, S2, CP, ldt, pst, p->ny, 0, sb, 0, h, p->nx, cap_th)))
      return rc;
    HFB_CUDA(cudaEventRecord(p->ov_ev[3], sb));
    y.mode = 0;
    y.src = S2;
    y.src_end = S2 + p->nz * pst;
    y.in_ld = ldt;
    ya = y;
    yb = y;
    ya.line0 = 0;
    ya.line1 = h;
    ya.max_per_sm = cap_dst;
    yb.line0 = h;
    yb.line1 = p->nx;
    HFB_CUDA(cudaStreamWaitEvent(st, p->ov_ev[2], 0));
    if ((rc = launch_dst16_mode(ya, st))) return rc;
    HFB_CUDA(cudaStreamWaitEvent(st, p->ov_ev[3], 0));
    mark(3);
    if ((rc = launch_dst16_mode(yb, st))) return rc;
    mark(4);
  } else {
    if ((rc = launch_dst16_mode(y, st))) return rc;
    mark(2);
    // 3
    if ((rc = fuse ? launch_thomas_tma(p, S2, CP, ldt, pst, st, 1)
                   : launch_thomas_tma_cached(p, S2, CP, ldt, pst, st)))
      return rc;
    mark(3);
    // 4
    y.mode = 0;
    y.src = S2;
    y.src_end = S2 + p->nz * pst;
    y.in_ld = ldt;
    if ((rc = launch_dst16_mode(y, st))) return rc;
    mark(4);
  }
  // 5
  x.mode = 2;
  x.src = S2;
  x.src_end = S2 + p->nz * pst;
  x.nrow = p->ny;
  x.in_ld = ldt;
  x.in_ps = pst;
  x.dst = out;
  x.out_ld = p->nx;
  x.out_ps = ps;
  if ((rc = launch_dst16_mode(x, st))) return rc;
  mark(5);
  return HFB_OK;
}

// Complex-coefficient solve (complex k(z)): the DSTs are real-linear, so the
// real and imaginary volumes are transformed separately by the same passes;
// the z-solve couples them. Fast layout: S1 + S2 (re) + S3 (im) + cp (two
// planes per chunk); lean: S2 + S3 + cp with transposing forward x-passes.
size_t fused_work_elems_z(const hfb_plan* p) {
  if (!tran_path(p)) return 0;
  const size_t nck = (p->nz + kThomasChunk - 1) / kThomasChunk;
  const size_t arrays = p->ws_lean ? 2 : 3;
  return (size_t)fused_plane(p) * (arrays * p->nz + 2 * nck);
}

static int forward_2d(hfb_plan* p, const double* rhs, double* S1, double* S2, cudaStream_t st) {
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), ldx = x_ld(p);
  const long long pst = fused_plane(p);
  if (dmma2d_np(p)) {  // small N: the DMMA whole-plane transform, as in solve_fused
    D2Layout fw = {p->nx, ps, ldt, pst, 0, 1};
    return launch_dmma2d(p, rhs, S2, 0, p->nz, st, &fw);
  }
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  Dst16Call y = x;
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  x.src = rhs;
  x.src_end = rhs + p->nz * ps;
  x.nrow = p->ny;
  x.in_ld = p->nx;
  x.in_ps = ps;
  x.mode = p->ws_lean ? 1 : 0;
  x.dst = p->ws_lean ? S2 : S1;
  x.out_ld = p->ws_lean ? ldt : ldx;
  x.out_ps = pst;
  int rc = launch_dst16_mode(x, st);
  if (rc) return rc;
  y.nrow = p->nx;
  y.dst = S2;
  y.out_ld = ldt;
  y.out_ps = pst;
  y.mode = p->ws_lean ? 0 : 2;
  y.src = p->ws_lean ? S2 : S1;
  y.in_ld = p->ws_lean ? ldt : ldx;
  y.src_end = y.src + p->nz * pst;
  y.in_ps = pst;
  return launch_dst16_mode(y, st);
}

static int inverse_2d(hfb_plan* p, double* S2, double* out, cudaStream_t st) {
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p);
  const long long pst = fused_plane(p);
  if (dmma2d_np(p)) {
    D2Layout iv = {ldt, pst, p->nx, ps, 1, 0};
    return launch_dmma2d(p, S2, out, 0, p->nz, st, &iv);
  }
  Dst16Call y = {};
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  y.nz = p->nz;
  Dst16Call x = y;
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  y.mode = 0;
  y.src = S2;
  y.src_end = S2 + p->nz * pst;
  y.nrow = p->nx;
  y.in_ld = ldt;
  y.in_ps = pst;
  y.dst = S2;
  y.out_ld = ldt;
  y.out_ps = pst;
  int rc = launch_dst16_mode(y, st);
  if (rc) return rc;
  x.mode = 2;
  x.src = S2;
  x.src_end = S2 + p->nz * pst;
  x.nrow = p->ny;
  x.in_ld = ldt;
  x.in_ps = pst;
  x.dst = out;
  x.out_ld = p->nx;
  x.out_ps = ps;
  return launch_dst16_mode(x, st);
}

int solve_fused_z(hfb_plan* p, const double* rhs_re, const double* rhs_im, double* out_re,
                  double* out_im, double* work, cudaStream_t st) {
  const long long pst = fused_plane(p), ldt = tran_ld(p);
  double* S1 = work;
  double* Sr = p->ws_lean ? work : work + pst * p->nz;
  double* Si = Sr + pst * p->nz;
  double* CP = Si + pst * p->nz;
  int rc;
  const StageMarks mark(p, st);
  mark(0);
  if ((rc = forward_2d(p, rhs_re, S1, Sr, st))) return rc;
  if ((rc = forward_2d(p, rhs_im, S1, Si, st))) return rc;
  mark(1);
  mark(2);
  if ((rc = launch_thomas_tma_z(p, Sr, Si, CP, ldt, pst, st))) return rc;
  mark(3);
  mark(4);
  if ((rc = inverse_2d(p, Sr, out_re, st))) return rc;
  if ((rc = inverse_2d(p, Si, out_im, st))) return rc;
  mark(5);
  return HFB_OK;
}

// Mode-space transforms for the partitioned solve (one rank's z-slab): the
// forward 2D DST writes padded mode rows (l, n, m) — the layout the exchange
// ships and the z-solve streams — and the inverse reads them back.
long long modes_ld(const hfb_plan* p) { return tran_ld(p); }
size_t modes_work_elems(const hfb_plan* p) {
  return tran_path(p) ? (size_t)p->nz * p->ny * x_ld(p) : 0;
}

int forward_modes(hfb_plan* p, const double* src, double* modes, double* S1, cudaStream_t st,
                  int parts, int kp) {
  if (!tran_path(p) || !S1) return HFB_ERR_ARGUMENT;
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), ldx = x_ld(p);
  if (dmma2d_np(p)) {  // small N: the one-call solve's DMMA transform (bitwise the same)
    if (parts > 0) return HFB_ERR_ARGUMENT;  // no packed output on this path
    D2Layout fw = {p->nx, ps, ldt, ldt * p->nx, 0, 1};
    return launch_dmma2d(p, src, modes, 0, p->nz, st, &fw);
  }
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  x.mode = 0;
  x.src = src;
  x.src_end = src + p->nz * ps;
  x.nrow = p->ny;
  x.in_ld = p->nx;
  x.in_ps = ps;
  x.dst = S1;
  x.out_ld = ldx;
  x.out_ps = ldx * p->ny;
  int rc = launch_dst16_mode(x, st);
  if (rc) return rc;
  Dst16Call y = {};
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  y.nz = p->nz;
  y.mode = 2;
  y.src = S1;
  y.src_end = S1 + p->nz * ldx * p->ny;
  y.nrow = p->nx;
  y.in_ld = ldx;
  y.in_ps = ldx * p->ny;
  y.dst = modes;
  y.out_ld = ldt;
  y.out_ps = ldt * p->nx;
  if (parts > 0) {
    // straight into the exchange blocks: block q = (n_z, n_x, kp), the line's
    // positions [q kp, (q + 1) kp) (modes is the send buffer)
    y.pack_parts = parts;
    y.pack_kp = kp;
    y.pack_bstride = (long long)p->nz * p->nx * kp;
  }
  return launch_dst16_mode(y, st);
}

int inverse_modes(hfb_plan* p, double* modes, double* out, cudaStream_t st) {
  if (!tran_path(p)) return HFB_ERR_ARGUMENT;
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), pst = ldt * p->nx;
  if (dmma2d_np(p)) {
    D2Layout iv = {ldt, pst, p->nx, ps, 1, 0};
    return launch_dmma2d(p, modes, out, 0, p->nz, st, &iv);
  }
  Dst16Call y = {};
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  y.nz = p->nz;
  y.mode = 0;
  y.src = modes;
  y.src_end = modes + p->nz * pst;
  y.nrow = p->nx;
  y.in_ld = ldt;
  y.in_ps = pst;
  y.dst = modes;
  y.out_ld = ldt;
  y.out_ps = pst;
  int rc = launch_dst16_mode(y, st);
  if (rc) return rc;
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  x.mode = 2;
  x.src = modes;
  x.src_end = modes + p->nz * pst;
  x.nrow = p->ny;
  x.in_ld = ldt;
  x.in_ps = pst;
  x.dst = out;
  x.out_ld = p->nx;
  x.out_ps = ps;
  return launch_dst16_mode(x, st);
}

int inverse_modes_blocks(hfb_plan* p, const double* back, double* modes, double* out, int parts,
                         int kp, cudaStream_t st) {
  if (!tran_path(p) || dmma2d_np(p) || parts < 1) return HFB_ERR_ARGUMENT;
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), pst = ldt * p->nx;
  Dst16Call y = {};
  y.tw = p->tw_y;
  y.sn = p->sn_y;
  y.scale = p->scale_y;
  y.M = p->ny + 1;
  y.nz = p->nz;
  y.mode = 0;
  y.src = back;  // rows gathered from the blocks by the row copies themselves
  y.src_end = back;
  y.nrow = p->nx;
  y.split_parts = parts;
  y.split_kp = kp;
  y.split_bstride = (long long)p->nz * p->nx * kp;
  y.dst = modes;
  y.out_ld = ldt;
  y.out_ps = pst;
  int rc = launch_dst16_mode(y, st);
  if (rc) return rc;
  Dst16Call x = {};
  x.tw = p->tw_x;
  x.sn = p->sn_x;
  x.scale = p->scale_x;
  x.M = p->nx + 1;
  x.nz = p->nz;
  x.mode = 2;
  x.src = modes;
  x.src_end = modes + p->nz * pst;
  x.nrow = p->ny;
  x.in_ld = ldt;
  x.in_ps = pst;
  x.dst = out;
  x.out_ld = p->nx;
  x.out_ps = ps;
  return launch_dst16_mode(x, st);
}

int transform_planes(hfb_plan* p, const double* src, double* dst, int z0, int z1, double* work,
                     cudaStream_t st) {
  const int nz = z1 - z0;
  if (nz <= 0) return HFB_OK;
  if (dmma2d_np(p)) return launch_dmma2d(p, src, dst, z0, z1, st);
  if (!tran_path(p) || force_dense(p)) {
    int rc = launch_dst_x(p, src, dst, z0, z1, 0, p->ny, work, st);
    if (rc) return rc;
    return launch_dst_y(p, dst, dst, z0, z1, 0, p->nx, work, st);
  }
  if (!work) return HFB_ERR_ARGUMENT;
  // x-pass: rows (l, j, :) -> scratch (l, n, j) ; y-pass: scratch lines
  // (l, n, :) -> natural (l, m, n). Scratch planes are indexed from 0.
  const long long ps = (long long)p->ny * p->nx, ldt = tran_ld(p), pst = ldt * p->nx;
  int rc = launch_dst16(p->tw_x, p->sn_x, p->scale_x, p->nx + 1, src + (long long)z0 * ps,
                        src + (long long)p->nz * ps, work, 0, nz, p->ny, p->nx, ps, ldt, pst,
                        true, st);
  if (rc) return rc;
  return launch_dst16(p->tw_y, p->sn_y, p->scale_y, p->ny + 1, work, work + nz * pst,
                      dst + (long long)z0 * ps, 0, nz, p->nx, ldt, pst, p->nx, ps, true, st);
}

}  // namespace hfb
