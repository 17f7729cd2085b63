// DST-I along contiguous lines with the register-resident engine (fft16.cuh),
// optionally writing the result transposed.
//
// A CTA holds NF transform groups; group f handles the line pair
// (r0 + 2f, r0 + 2f + 1) of one plane (pairs never straddle planes). Input
// lines are read straight from global memory in the cyclic order (a_e and
// its mirror a_{M-e}: the second read hits L1). Output:
//   ROW  : out[plane][row][pos]              (same line layout as the input)
//   TRAN : out[plane][pos][row]              (lines become columns: the
//          x-pass writes the y-pass's lines, the y-pass writes back the
//          natural (m, n) order). Staged through shared memory so each warp
//          store covers 2*NF consecutive rows of 8 positions.
#include <algorithm>

#include "fft16.cuh"

namespace hfb {

struct LinesArgs {
  const double* src;
  double* dst;
  int z0;          // first plane
  int nrow;        // lines per plane
  int ppp;         // line pairs per plane = ceil(nrow / 2)
  long long npairs;
  long long in_ld, in_ps;    // input: line stride, plane stride
  long long out_ld, out_ps;  // output: ROW: line stride; TRAN: position stride
  int N;           // line length = M - 1
  int NF;          // groups per CTA
  int stage_ld;    // TRAN staging row stride (odd, >= N)
};

template <bool TRAN>
__global__ void __launch_bounds__(256) dst16_lines_kernel(LinesArgs a, Fft16 c) {
  extern __shared__ double2 smem[];
  const int T = c.T;
  const int f = threadIdx.x / T, t = threadIdx.x - f * T;
  const int bufsz = pad16(c.M) + 1;
  double2* sb = smem + f * bufsz;
  double2* wsum = smem + a.NF * bufsz;
  const long long pair = (long long)blockIdx.x * a.NF + f;
  const bool live = pair < a.npairs;
  const long long pl = live ? a.z0 + pair / a.ppp : 0;
  const int r0 = live ? 2 * (int)(pair % a.ppp) : 0;
  const bool has1 = live && r0 + 1 < a.nrow;
  const double* in0 = a.src + pl * a.in_ps + (long long)r0 * a.in_ld - 1;  // a_e at in0[e]
  const double* in1 = in0 + a.in_ld;

  double2 v[16];
  dst16_pre(v, c, t, [&](int e) -> double2 {
    return make_double2(live ? __ldg(in0 + e) : 0.0, has1 ? __ldg(in1 + e) : 0.0);
  });
  fft16_forward(v, sb, c, t);
  double2 ev[8], od[8];
  dst16_post(v, sb, wsum, c, t, ev, od);

  if (!TRAN) {
    double* o0 = a.dst + pl * a.out_ps + (long long)r0 * a.out_ld;
    double* o1 = o0 + a.out_ld;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = t + T * i;
      if (live) {
        if (k >= 1) o0[2 * k - 1] = ev[i].x;
        o0[2 * k] = od[i].x;
      }
      if (has1) {
        if (k >= 1) o1[2 * k - 1] = ev[i].y;
        o1[2 * k] = od[i].y;
      }
    }
    return;
  }
  // TRAN: stage rows [2f, 2f+1] x positions into smem, then store columns.
  __syncthreads();  // every group is done with its FFT buffer
  double* st = reinterpret_cast<double*>(smem);
  double* s0 = st + (2 * f) * (long long)a.stage_ld;
  double* s1 = s0 + a.stage_ld;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = t + T * i;
    if (k >= 1) {
      s0[2 * k - 1] = ev[i].x;
      s1[2 * k - 1] = ev[i].y;
    }
    s0[2 * k] = od[i].x;
    s1[2 * k] = od[i].y;
  }
  __syncthreads();
  // CTA rows: pairs blockIdx.x*NF .. +NF-1 may span planes; store per row.
  const int W = 2 * a.NF;
  const long long total = (long long)a.N * W;
  for (long long e = threadIdx.x; e < total; e += blockDim.x) {
    const int pos = (int)(e / W), r = (int)(e - (long long)pos * W);
    const long long pr = (long long)blockIdx.x * a.NF + (r >> 1);
    if (pr >= a.npairs) continue;
    const long long plr = a.z0 + pr / a.ppp;
    const int row = 2 * (int)(pr % a.ppp) + (r & 1);
    if (row >= a.nrow) continue;
    a.dst[plr * a.out_ps + (long long)pos * a.out_ld + row] = st[r * (long long)a.stage_ld + pos];
  }
}

bool dst16_ok(int M) { return M >= 16 && M <= 4096 && (M & (M - 1)) == 0; }

// Lines (plane z0.., nrow lines each, line stride in_ld, plane stride in_ps)
// -> ROW (out_ld line stride) or TRAN (out_ld position stride).
int launch_dst16(const double2* tw, const double* sn, double scale, int M, const double* src,
                 double* dst, int z0, int nz, int nrow, long long in_ld, long long in_ps,
                 long long out_ld, long long out_ps, bool tran, cudaStream_t st) {
  if (nz <= 0 || nrow <= 0) return HFB_OK;
  Fft16 c;
  c.M = M;
  c.p = 0;
  while ((1 << c.p) < M) ++c.p;
  c.T = M / 16;
  c.tw = tw;
  c.sn = sn;
  c.scale = scale;
  LinesArgs a;
  a.src = src;
  a.dst = dst;
  a.z0 = z0;
  a.nrow = nrow;
  a.ppp = (nrow + 1) / 2;
  a.npairs = (long long)nz * a.ppp;
  a.in_ld = in_ld;
  a.in_ps = in_ps;
  a.out_ld = out_ld;
  a.out_ps = out_ps;
  a.N = M - 1;
  a.NF = std::max(1, std::min(256 / c.T, 8));
  while (a.NF * c.T < 32) ++a.NF;
  a.stage_ld = (a.N % 2 == 1) ? a.N + 2 : a.N + 1;  // odd stride: conflict-free columns
  const int threads = a.NF * c.T;
  const size_t fft_bytes = (size_t)a.NF * (pad16(M) + 1) * sizeof(double2);
  const size_t stage_bytes = tran ? (size_t)2 * a.NF * a.stage_ld * sizeof(double) : 0;
  const size_t sm = std::max(fft_bytes, stage_bytes) + (threads / 32 + 1) * sizeof(double2) +
                    sizeof(double2) * 2 * a.NF;
  const long long blocks = (a.npairs + a.NF - 1) / a.NF;
  if (tran) {
    HFB_CUDA(cudaFuncSetAttribute(dst16_lines_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dst16_lines_kernel<true><<<(unsigned)blocks, threads, sm, st>>>(a, c);
  } else {
    HFB_CUDA(cudaFuncSetAttribute(dst16_lines_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    dst16_lines_kernel<false><<<(unsigned)blocks, threads, sm, st>>>(a, c);
  }
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb
