// Register-resident DST-I engine for M = N+1 = 2^p, 16 <= M <= 4096.
//
// One transform group = T = M/16 threads; thread t holds the 16 complex
// values x[t + T*i] (the "cyclic" distribution). Stockham passes of radix 16
// (and one final radix 2/4/8 pass) run in registers; between passes the
// data is exchanged through a padded shared buffer (one pad slot per 16, so
// both the strided writes and the cyclic reads are bank-conflict free).
// The last pass leaves its outputs in the same cyclic slots, so the FFT
// needs (#passes - 1) exchanges: 2 for M = 512..4096.
//
// DST-I pre/post-processing (see hfb_internal.cuh for the algebra):
//   pre : b_e = s_e (a_e + a_{M-e}) + (a_e - a_{M-e})/2 from the loader;
//   post: B in registers -> C_k, D_k (k < M/2) with B_{M-k} read back from
//         shared memory; odd outputs are a prefix sum over k done on
//         contiguous k-segments (local scan + group scan), then handed back
//         in the cyclic order so every store of a warp is contiguous.
#pragma once
#include "hfb_internal.cuh"

namespace hfb {

__host__ __device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

// multiply by w16^e (forward: exp(-2 pi i e / 16)), e in 0..9 (compile time)
template <int E>
__device__ __forceinline__ double2 mul_w16(double2 a) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double r = 0.70710678118654752440;
  if (E == 0) return a;
  if (E == 4) return cmul_mi(a);
  if (E == 8) return make_double2(-a.x, -a.y);
  if (E == 2) return make_double2(r * (a.x + a.y), r * (a.y - a.x));
  if (E == 6) return make_double2(r * (a.y - a.x), -r * (a.x + a.y));
  // generic: w = (cos, -sin) of 2 pi E / 16
  const double wc = (E == 1) ? c1 : (E == 3) ? s1 : (E == 9) ? -c1 : 0.0;
  const double ws = (E == 1) ? s1 : (E == 3) ? c1 : (E == 9) ? -s1 : 0.0;
  // (a.x + i a.y)(wc - i ws)
  return make_double2(fma(a.x, wc, a.y * ws), fma(a.y, wc, -a.x * ws));
}

// in-place 16-point forward DFT of v[0..16) (4 x 4 decomposition)
__device__ __forceinline__ void dft16(double2* v) {
  double2 y[16];
#pragma unroll
  for (int u1 = 0; u1 < 4; ++u1) {
    double2 q[4] = {v[u1], v[u1 + 4], v[u1 + 8], v[u1 + 12]};
    dft_fwd<4>(q);
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) y[u1 * 4 + q2] = q[q2];
  }
  // twiddle y[u1][q2] *= w16^(u1*q2)
  y[1 * 4 + 1] = mul_w16<1>(y[5]);
  y[1 * 4 + 2] = mul_w16<2>(y[6]);
  y[1 * 4 + 3] = mul_w16<3>(y[7]);
  y[2 * 4 + 1] = mul_w16<2>(y[9]);
  y[2 * 4 + 2] = mul_w16<4>(y[10]);
  y[2 * 4 + 3] = mul_w16<6>(y[11]);
  y[3 * 4 + 1] = mul_w16<3>(y[13]);
  y[3 * 4 + 2] = mul_w16<6>(y[14]);
  y[3 * 4 + 3] = mul_w16<9>(y[15]);
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    double2 q[4] = {y[q2], y[4 + q2], y[8 + q2], y[12 + q2]};
    dft_fwd<4>(q);
#pragma unroll
    for (int q1 = 0; q1 < 4; ++q1) v[4 * q1 + q2] = q[q1];
  }
}

struct Fft16 {
  int M, p, T;                     // length, log2, threads per group
  const double2* __restrict__ tw;  // tw[k] = exp(-2 pi i k/M)
  const double* __restrict__ sn;   // sin(pi j/M), j <= M/2
  double scale;                    // sqrt(2/M)
};

// One radix-R Stockham pass on the cyclic registers (R in {2,4,8,16}).
// Butterflies j = t + T*b (b < 16/R) take slots b + u*(16/R).
template <int R>
__device__ __forceinline__ void pass_regs(double2* v, const Fft16& c, int L, int t) {
  constexpr int NB = 16 / R;
  const int twstep = c.M / (L * R);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + c.T * b;
    const int k = j & (L - 1);
    double2 w[R];
#pragma unroll
    for (int u = 0; u < R; ++u) w[u] = v[b + u * NB];
    if (L > 1) {
#pragma unroll
      for (int u = 1; u < R; ++u) w[u] = cmul(w[u], __ldg(&c.tw[u * k * twstep]));
    }
    if constexpr (R == 16) {
      dft16(w);
    } else {
      dft_fwd<R>(w);
    }
#pragma unroll
    for (int u = 0; u < R; ++u) v[b + u * NB] = w[u];
  }
}

// Write a pass's outputs (Stockham destination order) to shared memory.
template <int R>
__device__ __forceinline__ void pass_store(const double2* v, double2* sb, const Fft16& c, int L,
                                           int t) {
  constexpr int NB = 16 / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + c.T * b;
    const int k = j & (L - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int u = 0; u < R; ++u) sb[pad16(base + u * L)] = v[b + u * NB];
  }
}

__device__ __forceinline__ void load_cyclic(double2* v, const double2* sb, const Fft16& c, int t) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = sb[pad16(t + c.T * i)];
}

// Full forward FFT: v (cyclic, natural input order) -> v (cyclic, natural
// output order). sb: this group's padded buffer (>= pad16(M) slots). `bar`
// synchronises all groups of the CTA (every thread must call).
__device__ __forceinline__ void fft16_forward(double2* v, double2* sb, const Fft16& c, int t) {
  const int full = c.p / 4;     // radix-16 passes
  const int rem = c.p - 4 * full;  // final radix 2^rem (0 = none)
  int L = 1;
  for (int s = 0; s < full; ++s) {
    pass_regs<16>(v, c, L, t);
    const bool last = (s == full - 1) && rem == 0;
    if (!last) {
      pass_store<16>(v, sb, c, L, t);
      __syncthreads();
      load_cyclic(v, sb, c, t);
      __syncthreads();
    }
    L *= 16;
  }
  if (rem == 1) pass_regs<2>(v, c, L, t);
  else if (rem == 2) pass_regs<4>(v, c, L, t);
  else if (rem == 3) pass_regs<8>(v, c, L, t);
}

// Exclusive scan over the T threads of a group (T a power of two, groups
// are T-aligned runs of threadIdx.x). wsum: >= blockDim/32 slots.
__device__ __forceinline__ double2 group_scan16(double2 v, int t, int T, double2* wsum) {
  const int lane = threadIdx.x & 31;
  const int width = T < 32 ? T : 32;
  double2 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o < width) {
      const double tx = __shfl_up_sync(0xffffffffu, inc.x, o, width);
      const double ty = __shfl_up_sync(0xffffffffu, inc.y, o, width);
      if ((lane & (width - 1)) >= o) {
        inc.x += tx;
        inc.y += ty;
      }
    }
  }
  double2 ex = csub(inc, v);
  if (T > 32) {
    const int warp = threadIdx.x >> 5;
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    const int w0 = (threadIdx.x - t) >> 5;
    for (int w = w0; w < warp; ++w) ex = cadd(ex, wsum[w]);
  }
  return ex;
}

// DST post-processing. In: v = B (cyclic). Out: for i < 8 (k = t + T*i < M/2):
// ev[i] = sqrt(2/M) S_{2k} (= D_k; meaningless for k = 0) and od[i] =
// sqrt(2/M) S_{2k+1}. sb: group buffer; wsum: CTA scratch. M >= 16.
__device__ __forceinline__ void dst16_post(const double2* v, double2* sb, double2* wsum,
                                           const Fft16& c, int t, double2* ev, double2* od) {
  const int M = c.M, T = c.T;
#pragma unroll
  for (int i = 0; i < 16; ++i) sb[pad16(t + T * i)] = v[i];
  __syncthreads();
  double2 C[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = t + T * i;
    const double2 bk = v[i];
    const double2 bm = sb[pad16((M - k) & (M - 1))];
    C[i] = make_double2(0.5 * (bk.x + bm.x), 0.5 * (bk.y + bm.y));
    ev[i] = make_double2(-0.5 * c.scale * (bk.y - bm.y), 0.5 * c.scale * (bk.x - bm.x));
  }
  if (t == 0) C[0] = cscale(C[0], 0.5);
  __syncthreads();  // all B_{M-k} reads done before C overwrites the buffer
#pragma unroll
  for (int i = 0; i < 8; ++i) sb[pad16(t + T * i)] = C[i];
  __syncthreads();
  // contiguous segment k in [8t, 8t + 8): local inclusive scan
  double2 seg[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) seg[s] = sb[pad16(8 * t + s)];
#pragma unroll
  for (int s = 1; s < 8; ++s) seg[s] = cadd(seg[s], seg[s - 1]);
  const double2 off = group_scan16(seg[7], t, T, wsum);
  __syncthreads();  // segment reads (and wsum reads) done before P overwrites
#pragma unroll
  for (int s = 0; s < 8; ++s) sb[pad16(8 * t + s)] = cadd(seg[s], off);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) od[i] = cscale(sb[pad16(t + T * i)], c.scale);
}

// Pre-processing from a loader giving a_e for e in [1, M-1] (0 outside):
// v[i] = b_{t + T i}.
template <class Load>
__device__ __forceinline__ void dst16_pre(double2* v, const Fft16& c, int t, Load&& load) {
  const int M = c.M, T = c.T, H = M >> 1;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + T * i;
    if (e == 0) {
      v[i] = make_double2(0.0, 0.0);
    } else if (e == H) {
      const double2 a = load(e);
      v[i] = make_double2(2.0 * a.x, 2.0 * a.y);
    } else {
      const double2 p = load(e), q = load(M - e);
      const double s = __ldg(&c.sn[e < H ? e : M - e]);
      const double sx = (p.x + q.x) * s, sy = (p.y + q.y) * s;
      v[i] = make_double2(fma(0.5, p.x - q.x, sx), fma(0.5, p.y - q.y, sy));
    }
  }
}

}  // namespace hfb
