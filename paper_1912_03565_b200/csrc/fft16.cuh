// Register-resident DST-I engine for M = N+1 = 2^P, 16 <= M <= 4096, with the
// transform length a compile-time constant (all strides, twiddle steps and
// shared-memory padding fold to immediates).
//
// One transform group = T = M/16 threads; thread t holds the 16 complex
// values x[t + T*i] (the "cyclic" distribution). Stockham passes of radix 16
// (and one final radix 2/4/8 pass) run in registers; between passes the
// data is exchanged through a padded shared buffer (one pad slot per 16, so
// both the strided writes and the cyclic reads are bank-conflict free).
// The last pass leaves its outputs in the same cyclic slots, so the FFT
// needs (#passes - 1) exchanges: 2 for M = 512..4096.
//
// DST-I pre/post-processing (algebra in hfb_internal.cuh):
//   pre : b_e = s_e (a_e + a_{M-e}) + (a_e - a_{M-e})/2 from the loader;
//   post: B in registers -> C_k, D_k (k < M/2) with B_{M-k} read back from
//         shared memory; odd outputs are a prefix sum over k done on
//         contiguous k-segments (local scan + group scan), then handed back
//         in the cyclic order.
#pragma once
#include "hfb_internal.cuh"

namespace hfb {

__host__ __device__ __forceinline__ constexpr int pad16(int i) { return i + (i >> 4); }

// multiply by w16^E (forward: exp(-2 pi i E / 16))
template <int E>
__device__ __forceinline__ double2 mul_w16(double2 a) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double r = 0.70710678118654752440;
  if constexpr (E == 0) return a;
  if constexpr (E == 4) return cmul_mi(a);
  if constexpr (E == 2) return make_double2(r * (a.x + a.y), r * (a.y - a.x));
  if constexpr (E == 6) return make_double2(r * (a.y - a.x), -r * (a.x + a.y));
  constexpr double wc = (E == 1) ? c1 : (E == 3) ? s1 : -c1;  // E = 1, 3, 9
  constexpr double ws = (E == 1) ? s1 : (E == 3) ? c1 : -s1;
  return make_double2(fma(a.x, wc, a.y * ws), fma(a.y, wc, -a.x * ws));
}

// in-place 16-point forward DFT (4 x 4 decomposition)
__device__ __forceinline__ void dft16(double2* v) {
  double2 y[16];
#pragma unroll
  for (int u1 = 0; u1 < 4; ++u1) {
    double2 q[4] = {v[u1], v[u1 + 4], v[u1 + 8], v[u1 + 12]};
    dft_fwd<4>(q);
#pragma unroll
    for (int q2 = 0; q2 < 4; ++q2) y[u1 * 4 + q2] = q[q2];
  }
  y[5] = mul_w16<1>(y[5]);
  y[6] = mul_w16<2>(y[6]);
  y[7] = mul_w16<3>(y[7]);
  y[9] = mul_w16<2>(y[9]);
  y[10] = mul_w16<4>(y[10]);
  y[11] = mul_w16<6>(y[11]);
  y[13] = mul_w16<3>(y[13]);
  y[14] = mul_w16<6>(y[14]);
  y[15] = mul_w16<9>(y[15]);
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    double2 q[4] = {y[q2], y[4 + q2], y[8 + q2], y[12 + q2]};
    dft_fwd<4>(q);
#pragma unroll
    for (int q1 = 0; q1 < 4; ++q1) v[4 * q1 + q2] = q[q1];
  }
}

// Barrier over one transform group: a named barrier (id 1 + f, T threads)
// when the group is whole warps, else the CTA barrier.
template <int T>
__device__ __forceinline__ void group_sync(int f) {
  if constexpr (T >= 32) {
    asm volatile("bar.sync %0, %1;" ::"r"(f + 1), "n"(T) : "memory");
  } else {
    __syncthreads();
  }
}

template <int P>
struct F16 {
  static constexpr int M = 1 << P;
  static constexpr int T = M / 16;
  static constexpr int FULL = P / 4;
  static constexpr int REM = P % 4;
  static constexpr int BUF = pad16(M) + 1;  // double2 slots of a group buffer
};

// One radix-R Stockham pass (stride L) on the cyclic registers.
template <int P, int R, int L>
__device__ __forceinline__ void pass_regs(double2* v, const double2* __restrict__ tw, int t) {
  constexpr int M = F16<P>::M, T = F16<P>::T, NB = 16 / R, TWSTEP = M / (L * R);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j & (L - 1);
    double2 w[R];
#pragma unroll
    for (int u = 0; u < R; ++u) w[u] = v[b + u * NB];
    if constexpr (L > 1) {
#pragma unroll
      for (int u = 1; u < R; ++u) w[u] = cmul(w[u], __ldg(&tw[u * k * TWSTEP]));
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

// Store the outputs of a radix-16 pass in Stockham order, then reload cyclic.
template <int P, int L>
__device__ __forceinline__ void exchange16(double2* v, double2* sb, int t, int f) {
  constexpr int T = F16<P>::T;
  const int k = t & (L - 1);
  const int base = (t - k) * 16 + k;
#pragma unroll
  for (int u = 0; u < 16; ++u) sb[pad16(base + u * L)] = v[u];
  group_sync<T>(f);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = sb[pad16(t + T * i)];
  group_sync<T>(f);
}

// Full forward FFT: cyclic natural-order input -> cyclic natural-order output.
template <int P>
__device__ __forceinline__ void fft16_forward(double2* v, double2* sb,
                                              const double2* __restrict__ tw, int t, int f) {
  using G = F16<P>;
  pass_regs<P, 16, 1>(v, tw, t);
  if constexpr (G::FULL >= 2) {
    exchange16<P, 1>(v, sb, t, f);
    pass_regs<P, 16, 16>(v, tw, t);
  }
  if constexpr (G::FULL >= 3) {
    exchange16<P, 16>(v, sb, t, f);
    pass_regs<P, 16, 256>(v, tw, t);
  }
  if constexpr (G::REM > 0) {
    constexpr int L = 1 << (4 * G::FULL);
    exchange16<P, L / 16>(v, sb, t, f);
    pass_regs<P, (1 << G::REM), L>(v, tw, t);
  }
}

// Exclusive scan over the T threads of a group (T-aligned runs of threadIdx).
template <int T>
__device__ __forceinline__ double2 group_scan(double2 v, int t, int f, double2* wsum) {
  constexpr int W = T < 32 ? T : 32;
  const int lane = threadIdx.x & 31;
  double2 inc = v;
#pragma unroll
  for (int o = 1; o < W; o <<= 1) {
    const double tx = __shfl_up_sync(0xffffffffu, inc.x, o, W);
    const double ty = __shfl_up_sync(0xffffffffu, inc.y, o, W);
    if ((lane & (W - 1)) >= o) {
      inc.x += tx;
      inc.y += ty;
    }
  }
  double2 ex = csub(inc, v);
  if constexpr (T > 32) {
    const int warp = threadIdx.x >> 5;
    if (lane == 31) wsum[warp] = inc;
    group_sync<T>(f);
    const int w0 = (threadIdx.x - t) >> 5;
#pragma unroll
    for (int w = 0; w < T / 32 - 1; ++w)
      if (w0 + w < warp) ex = cadd(ex, wsum[w0 + w]);
  }
  return ex;
}

// DST post-processing. In: v = B (cyclic). Out: for i < 8 (k = t + T i):
// ev[i] = scale * S_{2k} (D_k; unused for k = 0), od[i] = scale * S_{2k+1}.
template <int P>
__device__ __forceinline__ void dst16_post(const double2* v, double2* sb, double2* wsum,
                                           double scale, int t, int f, double2* ev,
                                           double2* od) {
  constexpr int M = F16<P>::M, T = F16<P>::T;
#pragma unroll
  for (int i = 0; i < 16; ++i) sb[pad16(t + T * i)] = v[i];
  group_sync<T>(f);
  double2 C[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = t + T * i;
    const double2 bk = v[i];
    const double2 bm = sb[pad16((M - k) & (M - 1))];
    C[i] = make_double2(0.5 * (bk.x + bm.x), 0.5 * (bk.y + bm.y));
    ev[i] = make_double2(-0.5 * scale * (bk.y - bm.y), 0.5 * scale * (bk.x - bm.x));
  }
  if (t == 0) C[0] = cscale(C[0], 0.5);
  group_sync<T>(f);
#pragma unroll
  for (int i = 0; i < 8; ++i) sb[pad16(t + T * i)] = C[i];
  group_sync<T>(f);
  double2 seg[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) seg[s] = sb[pad16(8 * t + s)];
#pragma unroll
  for (int s = 1; s < 8; ++s) seg[s] = cadd(seg[s], seg[s - 1]);
  const double2 off = group_scan<T>(seg[7], t, f, wsum);
  group_sync<T>(f);
#pragma unroll
  for (int s = 0; s < 8; ++s) sb[pad16(8 * t + s)] = cadd(seg[s], off);
  group_sync<T>(f);
#pragma unroll
  for (int i = 0; i < 8; ++i) od[i] = cscale(sb[pad16(t + T * i)], scale);
}

// Pre-processing: v[i] = b_{t + T i} from a loader of a_e (e in [1, M-1]); the
// loader may return garbage for e = 0 and e = M (selected away here). The one
// formula also covers b_0 = 0 (s_0 = 0, a_0 = a_M = 0) and b_{M/2} = 2 a_{M/2}.
template <int P, class Load>
__device__ __forceinline__ void dst16_pre(double2* v, const double* __restrict__ sn, int t,
                                          Load&& load) {
  constexpr int M = F16<P>::M, T = F16<P>::T, H = M / 2;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + T * i;
    double2 p = load(e), q = load(M - e);
    if (i == 0) {
      const bool z = (t == 0);
      p = z ? make_double2(0.0, 0.0) : p;
      q = z ? make_double2(0.0, 0.0) : q;
    }
    const double s = __ldg(&sn[e <= H ? e : M - e]);
    const double sx = (p.x + q.x) * s, sy = (p.y + q.y) * s;
    v[i] = make_double2(fma(0.5, p.x - q.x, sx), fma(0.5, p.y - q.y, sy));
  }
}

}  // namespace hfb
