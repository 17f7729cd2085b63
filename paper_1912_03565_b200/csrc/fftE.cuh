// Register-resident DST-I engine, E = 16 or 32 complex values per thread,
// transform length M = N+1 = 2^P a compile-time constant (E <= M <= 4096).
//
// A transform group = T = M/E threads; thread t holds x[t + T*i], i < E (the
// "cyclic" distribution). Stockham passes of radix E (and one final smaller
// radix) run in registers; between passes the values go through a shared
// buffer whose slots are XOR-swizzled (swz), so the strided Stockham writes and
// the cyclic reads are bank-conflict free without padding. The last pass
// leaves its outputs in the same cyclic slots: an M = 1024 transform with
// E = 32 is one warp, two radix-32 passes and a single exchange.
//
// DST-I pre/post-processing (algebra in hfb_internal.cuh):
//   pre : b_e = s_e (a_e + a_{M-e}) + (a_e - a_{M-e})/2 (b_0 = 0 and
//         b_{M/2} = 2 a_{M/2} fall out of the same formula);
//   post: B goes to shared memory once; thread t then reads its contiguous
//         k-segment [SEG t, SEG t + SEG) (SEG = E/2) together with the mirror
//         values B_{M-k}, forms C_k and D_k, scans C over the segment and the
//         segment totals over the group, and emits the 2 SEG consecutive
//         outputs S_{2k} (position 2k-1) and S_{2k+1} (position 2k).
#pragma once
#include "hfb_internal.cuh"

namespace hfb {

// cos(pi k / 16) for any integer k (exact decimal expansions of the 32nd roots)
__host__ __device__ __forceinline__ constexpr double c32(int k) {
  constexpr double tab[9] = {1.0,
                             0.98078528040323044913,
                             0.92387953251128675613,
                             0.83146961230254523708,
                             0.70710678118654752440,
                             0.55557023301960222474,
                             0.38268343236508977173,
                             0.19509032201612826785,
                             0.0};
  const int m = ((k % 32) + 32) % 32;
  return m <= 8 ? tab[m] : m <= 16 ? -tab[16 - m] : m <= 24 ? -tab[m - 16] : tab[32 - m];
}

// HFB_CONST_BANK: the same cosines from a __constant__ table, so the FP64
// instructions take them as constant-bank operands instead of 64-bit
// immediates moved through uniform registers (two UMOV each).
#ifndef HFB_CONST_BANK
#define HFB_CONST_BANK 0
#endif
#if HFB_CONST_BANK
__constant__ double kC32[9] = {1.0,
                               0.98078528040323044913,
                               0.92387953251128675613,
                               0.83146961230254523708,
                               0.70710678118654752440,
                               0.55557023301960222474,
                               0.38268343236508977173,
                               0.19509032201612826785,
                               0.0};
__device__ __forceinline__ double c32v(int k) {  // k a compile-time constant after unrolling
  const int m = ((k % 32) + 32) % 32;
  return m <= 8 ? kC32[m] : m <= 16 ? -kC32[16 - m] : m <= 24 ? -kC32[m - 16] : kC32[32 - m];
}
#else
__device__ __forceinline__ constexpr double c32v(int k) { return c32(k); }
#endif

// multiply by w_N^E = exp(-2 pi i E / N) for a compile-time (N, E), N | 32
template <int N, int E>
__device__ __forceinline__ double2 mul_wn(double2 a) {
  constexpr int e = ((E % N) + N) % N;
  const double r = c32v(4);
  if constexpr (e == 0) {
    return a;
  } else if constexpr (4 * e == N) {  // -i
    return cmul_mi(a);
  } else if constexpr (2 * e == N) {  // -1
    return make_double2(-a.x, -a.y);
  } else if constexpr (4 * e == 3 * N) {  // +i
    return make_double2(-a.y, a.x);
  } else if constexpr (8 * e == N) {  // (1 - i)/sqrt2
    return make_double2(r * (a.x + a.y), r * (a.y - a.x));
  } else if constexpr (8 * e == 3 * N) {  // (-1 - i)/sqrt2
    return make_double2(r * (a.y - a.x), -r * (a.x + a.y));
  } else {
    constexpr int K = e * (32 / N);  // angle 2 pi e / N = pi K / 16
    const double wc = c32v(K), ws = c32v(K - 8);  // cos, sin
    return make_double2(fma(a.x, wc, a.y * ws), fma(a.y, wc, -a.x * ws));
  }
}

// in-place forward DFT of R values (natural order in and out)
template <int R>
__device__ __forceinline__ void dftR(double2* v);

template <>
__device__ __forceinline__ void dftR<2>(double2* v) {
  dft_fwd<2>(v);
}
template <>
__device__ __forceinline__ void dftR<4>(double2* v) {
  dft_fwd<4>(v);
}
template <>
__device__ __forceinline__ void dftR<8>(double2* v) {
  dft_fwd<8>(v);
}

// R = N1 * N2 split: u = u1 + N1 u2, q = N2 q1 + q2
template <int N1, int N2>
__device__ __forceinline__ void dft_split(double2* v) {
  constexpr int R = N1 * N2;
  double2 y[R];
#pragma unroll
  for (int u1 = 0; u1 < N1; ++u1) {
    double2 q[N2];
#pragma unroll
    for (int u2 = 0; u2 < N2; ++u2) q[u2] = v[u1 + N1 * u2];
    dftR<N2>(q);
#pragma unroll
    for (int q2 = 0; q2 < N2; ++q2) y[u1 * N2 + q2] = q[q2];
  }
  // twiddle y[u1][q2] *= w_R^(u1 q2)
#pragma unroll
  for (int u1 = 1; u1 < N1; ++u1) {
#pragma unroll
    for (int q2 = 1; q2 < N2; ++q2) {
      // unrolled constant exponent via a switch on the product
      double2& z = y[u1 * N2 + q2];
      switch (u1 * q2) {
#define HFB_TW(EE) \
  case EE: z = mul_wn<R, EE>(z); break;
        HFB_TW(1) HFB_TW(2) HFB_TW(3) HFB_TW(4) HFB_TW(5) HFB_TW(6) HFB_TW(7) HFB_TW(8)
        HFB_TW(9) HFB_TW(10) HFB_TW(12) HFB_TW(14) HFB_TW(15) HFB_TW(18) HFB_TW(21)
#undef HFB_TW
        default: break;
      }
    }
  }
#pragma unroll
  for (int q2 = 0; q2 < N2; ++q2) {
    double2 q[N1];
#pragma unroll
    for (int u1 = 0; u1 < N1; ++u1) q[u1] = y[u1 * N2 + q2];
    dftR<N1>(q);
#pragma unroll
    for (int q1 = 0; q1 < N1; ++q1) v[N2 * q1 + q2] = q[q1];
  }
}

template <>
__device__ __forceinline__ void dftR<16>(double2* v) {
  dft_split<4, 4>(v);
}
template <>
__device__ __forceinline__ void dftR<32>(double2* v) {
  dft_split<4, 8>(v);
}

template <int T>
__device__ __forceinline__ void group_sync(int f) {
  if constexpr (T == 32) {
    __syncwarp();
  } else if constexpr (T > 32) {
    asm volatile("bar.sync %0, %1;" ::"r"(f + 1), "n"(T) : "memory");
  } else {
    __syncthreads();
  }
}

template <int P, int E>
struct FE {
  static constexpr int M = 1 << P;
  static constexpr int T = M / E;
  static constexpr int LE = (E == 32) ? 5 : 4;
  static constexpr int FULL = P / LE;
  static constexpr int REM = P % LE;
  static constexpr int SEG = E / 2;
  static constexpr int BUF = M;  // double2 slots of a group buffer (XOR-swizzled, no pads)
};

// Bank-conflict-free placement without padding: the low three bits of a
// 16-byte slot index are XORed with bits [S, S+3). Accesses whose threads
// stride by 2^S slots (the Stockham scatter, the k-segment reads of the post-
// processing) and accesses by 8 consecutive slots both hit 8 distinct bank
// groups, and the map is a bijection inside every aligned block of 8 slots.
template <int S>
__device__ __forceinline__ constexpr int swz(int i) {
  return i ^ ((i >> S) & 7);
}

// Shared-memory accesses by 32-bit shared address. For groups of whole warps
// (T >= 32) the launch code keeps every group buffer 256-byte aligned, so a
// swizzled slot "base ^ column" is one XOR on the byte address (no separate
// index-to-address step). volatile keeps these in program order with the
// group barriers (also volatile asm); the stores clobber memory.
__device__ __forceinline__ uint32_t sh_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void sh_st2(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
template <int OFF>
__device__ __forceinline__ void sh_st2_off(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0+%3], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y), "n"(OFF)
               : "memory");
}
__device__ __forceinline__ double2 sh_ld2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
#ifndef HFB_XOR_ADDR
#define HFB_XOR_ADDR 1  // 0: index forms everywhere (A/B builds)
#endif
template <int P, int E>
constexpr bool kXorAddr = (HFB_XOR_ADDR && E == 16 && FE<P, E>::T >= 32);

// multiply by w_N^e for an e that is a compile-time constant after unrolling
template <int N>
__device__ __forceinline__ double2 mul_wn_at(double2 a, int e) {
  switch (e & 31) {
#define HFB_W(EE) \
  case EE: return mul_wn<N, EE>(a);
    HFB_W(0) HFB_W(1) HFB_W(2) HFB_W(3) HFB_W(4) HFB_W(5) HFB_W(6) HFB_W(7) HFB_W(8) HFB_W(9)
    HFB_W(10) HFB_W(11) HFB_W(12) HFB_W(13) HFB_W(14) HFB_W(15) HFB_W(16) HFB_W(17) HFB_W(18)
    HFB_W(19) HFB_W(20) HFB_W(21) HFB_W(22) HFB_W(23) HFB_W(24) HFB_W(25) HFB_W(26) HFB_W(27)
    HFB_W(28) HFB_W(29) HFB_W(30) HFB_W(31)
#undef HFB_W
  }
  return a;
}

// Per-thread twiddle bases, loaded once per kernel (they depend only on the
// thread's place in its group, not on the data): for the pass of stride L and
// radix R, w = tw[k M/(L R)] with k = t mod L, plus w^4 (R >= 16) and w^16
// (R = 32) straight from the table; the sine pair of the pre-processing.
template <int P, int E>
struct EngineTw {
  double2 w1[3], w4[3], w16[3];  // by pass index (0 = the L = 1 pass: unused)
  double st, ct;                 // sin(pi t/M), cos(pi t/M)
};

template <int P, int E, int R, int L>
__device__ __forceinline__ void tw_base(const double2* __restrict__ tw, int t, double2& w1,
                                        double2& w4, double2& w16) {
  constexpr int M = FE<P, E>::M, TWSTEP = M / (L * R);
  const int k = t & (L - 1);
  w1 = __ldg(&tw[k * TWSTEP]);
  if constexpr (R >= 16) w4 = __ldg(&tw[4 * k * TWSTEP]);
  if constexpr (R == 32) w16 = __ldg(&tw[16 * k * TWSTEP]);
}

template <int P, int E>
__device__ __forceinline__ void engine_tw(const double2* __restrict__ tw,
                                          const double* __restrict__ sn, int t,
                                          EngineTw<P, E>& w) {
  using G = FE<P, E>;
  if constexpr (G::FULL >= 2) tw_base<P, E, E, E>(tw, t, w.w1[1], w.w4[1], w.w16[1]);
  if constexpr (G::FULL >= 3) tw_base<P, E, E, E * E>(tw, t, w.w1[2], w.w4[2], w.w16[2]);
  if constexpr (G::REM > 0) {
    constexpr int L = 1 << (G::LE * G::FULL);
    tw_base<P, E, (1 << G::REM), L>(tw, t, w.w1[G::FULL], w.w4[G::FULL], w.w16[G::FULL]);
  }
  w.st = __ldg(&sn[t]);
  w.ct = __ldg(&sn[G::M / 2 - t]);
}

// Twiddles w^u, u = 1..R-1, from w (and w^4, w^16 for R >= 16, 32): w^2, w^3
// by products, so every factor is at most four roundings from the table.
template <int R>
__device__ __forceinline__ void twiddle_powers(double2 w1, double2 w4, double2 w16,
                                               double2* wp) {
  wp[1] = w1;
  if constexpr (R >= 4) {
    wp[2] = cmul(wp[1], wp[1]);
    wp[3] = cmul(wp[2], wp[1]);
  }
  if constexpr (R == 8) {
    wp[4] = cmul(wp[2], wp[2]);
    wp[5] = cmul(wp[4], wp[1]);
    wp[6] = cmul(wp[4], wp[2]);
    wp[7] = cmul(wp[4], wp[3]);
  }
  if constexpr (R >= 16) {
    wp[4] = w4;
    wp[8] = cmul(wp[4], wp[4]);
    wp[12] = cmul(wp[8], wp[4]);
#pragma unroll
    for (int a4 = 4; a4 < 16; a4 += 4)
#pragma unroll
      for (int b = 1; b < 4; ++b) wp[a4 + b] = cmul(wp[a4], wp[b]);
  }
  if constexpr (R == 32) {
    wp[16] = w16;
#pragma unroll
    for (int r = 1; r < 16; ++r) wp[16 + r] = cmul(wp[16], wp[r]);
  }
}

// One radix-R Stockham pass (stride L) on the cyclic registers. With NB = E/R
// butterflies per thread (the final, smaller-radix pass), butterfly b's base
// is tw[t + T b] = w * w_E^b: one rotation by a compile-time root.
template <int P, int E, int R, int L>
__device__ __forceinline__ void pass_regs(double2* v, double2 w1, double2 w4, double2 w16) {
  constexpr int NB = E / R;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double2 w[R];
#pragma unroll
    for (int u = 0; u < R; ++u) w[u] = v[b + u * NB];
    if constexpr (L > 1) {
      static_assert(NB == 1 || FE<P, E>::T * NB == L, "shared twiddle base");
      const double2 b1 = b ? mul_wn_at<E>(w1, b) : w1;
      const double2 b4 = b ? mul_wn_at<E>(w4, 4 * b) : w4;
      const double2 b16 = b ? mul_wn_at<E>(w16, 16 * b) : w16;
      if constexpr (R >= 16) {
        // w^(4a + c) = w^(4a) w^c generated as they are used (the values of
        // twiddle_powers, without holding all R - 1 powers live); for R = 32
        // w^(16 + u) = w^16 w^u in the same step
        const double2 p2 = cmul(b1, b1), p3 = cmul(p2, b1);
        double2 q = b4;
#pragma unroll
        for (int a4 = 0; a4 < 4; ++a4) {
          if (a4 == 2) q = cmul(b4, b4);
          if (a4 == 3) q = cmul(q, b4);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int u = 4 * a4 + c;
            double2 f;
            if (u == 0) {
              if constexpr (R == 32) w[16] = cmul(w[16], b16);
              continue;
            } else if (a4 == 0) {
              f = c == 1 ? b1 : c == 2 ? p2 : p3;
            } else {
              f = c == 0 ? q : cmul(q, c == 1 ? b1 : c == 2 ? p2 : p3);
            }
            w[u] = cmul(w[u], f);
            if constexpr (R == 32) w[u + 16] = cmul(w[u + 16], cmul(b16, f));
          }
        }
      } else {
        double2 wp[R];
        twiddle_powers<R>(b1, b4, b16, wp);
#pragma unroll
        for (int u = 1; u < R; ++u) w[u] = cmul(w[u], wp[u]);
      }
    }
    dftR<R>(w);
#pragma unroll
    for (int u = 0; u < R; ++u) v[b + u * NB] = w[u];
  }
}

// Swizzled slot of the cyclic element t + T i in closed form (S = LE or LE - 1,
// T a multiple of 2^S): the XOR term ((t >> S) + (T >> S) i) & 7 takes at most
// 8 / gcd(8, T >> S) values over i, so the slots are a few per-thread bases plus
// compile-time offsets T i (base + immediate addressing, no per-element
// integer arithmetic; the same slots as swz<S>(t + T i)).
template <int T, int S>
struct CyclicSlots {
  static constexpr int STEP = (T >> S) & 7;
  static constexpr int NC = STEP == 0 ? 1 : (STEP & 1) ? 8 : (STEP & 2) ? 4 : 2;
  int base[NC];
  __device__ __forceinline__ explicit CyclicSlots(int t) {
    static_assert(T >= (1 << S) && T >= 8, "closed form needs T >= max(8, 2^S)");
    const int a = (t >> S) & 7;
#pragma unroll
    for (int c = 0; c < NC; ++c) base[c] = t ^ ((a + STEP * c) & 7);
  }
  __device__ __forceinline__ int at(int i) const { return base[i % NC] + T * i; }
};

// Store a radix-E pass's outputs in Stockham order, then reload cyclic.
template <int P, int E, int L>
__device__ __forceinline__ void exchangeE(double2* v, double2* sb, int t, int f) {
  constexpr int T = FE<P, E>::T;
  constexpr int LE = FE<P, E>::LE;
  const int k = t & (L - 1);
  const int base = (t - k) * E + k;
  if constexpr (E == 16 && L == 1) {
    // slot 16 t + u, XOR term t & 7: (16 t ^ (t & 7)) ^ u
    const int b0 = (16 * t) ^ (t & 7);
    if constexpr (kXorAddr<P, E>) {
      const uint32_t a0 = sh_addr(sb) + 16u * (uint32_t)b0;
#pragma unroll
      for (int u = 0; u < E; ++u) sh_st2(a0 ^ (16u * u), v[u]);
    } else {
#pragma unroll
      for (int u = 0; u < E; ++u) sb[b0 ^ u] = v[u];
    }
  } else if constexpr (E == 16 && L == 16) {
    // slot base + 16 u with base = 16 (t - k) + k, k < 16: XOR term u & 7 on
    // k's low bits: (base ^ (u & 7)) + 16 u
    if constexpr (kXorAddr<P, E>) {
      const uint32_t a0 = sh_addr(sb) + 16u * (uint32_t)base;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t au = a0 ^ (16u * u);
        sh_st2(au + 256u * u, v[u]);
        sh_st2(au + 256u * (u + 8), v[u + 8]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < E; ++u) sb[(base ^ (u & 7)) + u * L] = v[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < E; ++u) sb[swz<LE>(base + u * L)] = v[u];
  }
  group_sync<T>(f);
  if constexpr (E == 16 && T >= 16) {
    const CyclicSlots<T, LE> cs(t);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = sb[cs.at(i)];
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = sb[swz<LE>(t + T * i)];
  }
  group_sync<T>(f);
}

template <int P, int E>
__device__ __forceinline__ void fftE_forward(double2* v, double2* sb, const EngineTw<P, E>& tw,
                                             int t, int f) {
  using G = FE<P, E>;
  const double2 z = make_double2(0.0, 0.0);
  pass_regs<P, E, E, 1>(v, z, z, z);
  if constexpr (G::FULL >= 2) {
    exchangeE<P, E, 1>(v, sb, t, f);
    pass_regs<P, E, E, E>(v, tw.w1[1], tw.w4[1], tw.w16[1]);
  }
  if constexpr (G::FULL >= 3) {
    exchangeE<P, E, E>(v, sb, t, f);
    pass_regs<P, E, E, E * E>(v, tw.w1[2], tw.w4[2], tw.w16[2]);
  }
  if constexpr (G::REM > 0) {
    constexpr int L = 1 << (G::LE * G::FULL);
    exchangeE<P, E, L / E>(v, sb, t, f);
    pass_regs<P, E, (1 << G::REM), L>(v, tw.w1[G::FULL], tw.w4[G::FULL], tw.w16[G::FULL]);
  }
}

// Exclusive scan over the T threads of a group (T-aligned runs of threadIdx).
template <int T>
__device__ __forceinline__ double2 group_scanE(double2 v, int t, int f, double2* wsum) {
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

// Post-processing slots (swizzle S = LE - 1, SEG = 2^S values per thread).
// post_store: B_{t + T i} at swz<S>(t + T i). PostSlots: thread t's segment
// values B_k, k = SEG t + s (s <= SEG), and their mirrors B_{(M - k) mod M}, at
// swz<S>(.) — for E = 16 in closed form: k and M - k stay inside one 8-slot row
// for s in [0, 8) resp. [1, 8], where the XOR term is the row's low bits, so a
// slot is (row base ^ row bits) ^ column: one XOR with a compile-time column.
template <int P, int E>
__device__ __forceinline__ void post_store(const double2* v, double2* sb, int t) {
  constexpr int T = FE<P, E>::T, LS = FE<P, E>::LE - 1;
  if constexpr (E == 16 && T >= 8) {
    const CyclicSlots<T, LS> cs(t);
#pragma unroll
    for (int i = 0; i < E; ++i) sb[cs.at(i)] = v[i];
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) sb[swz<LS>(t + T * i)] = v[i];
  }
}

template <int P, int E>
struct PostSlots {
  static constexpr int M = FE<P, E>::M, SEG = FE<P, E>::SEG, LS = FE<P, E>::LE - 1;
  static constexpr bool FAST = (E == 16);
  int t, f0, f1, m0, m1;
  __device__ __forceinline__ explicit PostSlots(int tt) : t(tt) {
    if constexpr (FAST) {
      const int R = M / 8;  // 8-slot rows of the buffer
      f0 = (8 * t) ^ (t & 7);                    // row t: k = 8 t + s, s < 8
      f1 = (8 * (t + 1)) ^ ((t + 1) & 7);        // k = 8 (t + 1) <= M/2
      const int r0 = (R - t) & (R - 1);          // M - 8 t (mod M) = 8 r0
      m0 = (8 * r0) ^ (r0 & 7);
      const int r1 = R - 1 - t;                  // M - 8 t - s = 8 r1 + (8 - s), 1 <= s <= 8
      m1 = (8 * r1) ^ (r1 & 7);
    }
  }
  // byte-address forms (128-byte aligned buffer at shared address a)
  __device__ __forceinline__ uint32_t fwd_addr(uint32_t a, int s) const {
    return s < 8 ? ((a + 16u * (uint32_t)f0) ^ (16u * s)) : a + 16u * (uint32_t)f1;
  }
  __device__ __forceinline__ uint32_t mir_addr(uint32_t a, int s) const {
    return s == 0 ? a + 16u * (uint32_t)m0 : ((a + 16u * (uint32_t)m1) ^ (16u * (8 - s)));
  }
  __device__ __forceinline__ int fwd(int s) const {
    if constexpr (FAST) return s < 8 ? (f0 ^ s) : f1;
    return swz<LS>((SEG * t + s) & (M - 1));
  }
  __device__ __forceinline__ int mir(int s) const {
    if constexpr (FAST) return s == 0 ? m0 : (m1 ^ (8 - s));
    return swz<LS>((M - SEG * t - s) & (M - 1));
  }
};

// DST post-processing: v = B (cyclic) -> the 2*SEG outputs of thread t, i.e.
// positions 2k-1 and 2k for k in [SEG t, SEG t + SEG), scaled by sqrt(2/M):
// out[2s] = S_{2k} (position 2k-1; meaningless for k = 0), out[2s+1] =
// S_{2k+1} (position 2k), k = SEG t + s. sb is left free for the caller.
template <int P, int E>
__device__ __forceinline__ void dstE_post(const double2* v, double2* sb, double2* wsum,
                                          double scale, int t, int f, double2* out) {
  constexpr int M = FE<P, E>::M, T = FE<P, E>::T, SEG = FE<P, E>::SEG, LS = FE<P, E>::LE - 1;
  post_store<P, E>(v, sb, t);
  group_sync<T>(f);
  const int k0 = SEG * t;
  const PostSlots<P, E> ps(t);
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s < SEG; ++s) {
    const int k = k0 + s;
    double2 bk, bm;
    if constexpr (kXorAddr<P, E>) {
      bk = sh_ld2(ps.fwd_addr(sh_addr(sb), s));
      bm = sh_ld2(ps.mir_addr(sh_addr(sb), s));
    } else {
      bk = sb[ps.fwd(s)];
      bm = sb[ps.mir(s)];
    }
    double2 C = make_double2(0.5 * (bk.x + bm.x), 0.5 * (bk.y + bm.y));
    if (k == 0) C = cscale(C, 0.5);
    run = cadd(run, C);
    out[2 * s] = make_double2(-0.5 * scale * (bk.y - bm.y), 0.5 * scale * (bk.x - bm.x));
    out[2 * s + 1] = run;  // inclusive prefix within the segment (unscaled)
  }
  const double2 off = group_scanE<T>(run, t, f, wsum);
#pragma unroll
  for (int s = 0; s < SEG; ++s) out[2 * s + 1] = cscale(cadd(out[2 * s + 1], off), scale);
  group_sync<T>(f);  // every B read is done: sb may be reused
}

// Post-processing with segment-aligned ownership: thread t emits positions
// [Q t, Q t + Q) (Q = 2 SEG) — out[2s] = S_{2k+1} (position 2k) and
// out[2s+1] = S_{2k+2} = D_{k+1} (position 2k+1), k = SEG t + s — so every
// thread owns whole 128-byte segments of the output line (for TMA tensor
// stores). Costs one extra (B_k, B_{M-k}) read per thread for D_{SEG t + SEG}.
template <int P, int E>
__device__ __forceinline__ void dstE_post_aligned(const double2* v, double2* sb, double2* wsum,
                                                  double scale, int t, int f, double2* out) {
  constexpr int M = FE<P, E>::M, T = FE<P, E>::T, SEG = FE<P, E>::SEG, LS = FE<P, E>::LE - 1;
  post_store<P, E>(v, sb, t);
  group_sync<T>(f);
  const int k0 = SEG * t;
  const PostSlots<P, E> ps(t);
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int s = 0; s <= SEG; ++s) {
    const int k = k0 + s;  // k <= M/2
    double2 bk, bm;
    if constexpr (kXorAddr<P, E>) {
      bk = sh_ld2(ps.fwd_addr(sh_addr(sb), s));
      bm = sh_ld2(ps.mir_addr(sh_addr(sb), s));
    } else {
      bk = sb[ps.fwd(s)];
      bm = sb[ps.mir(s)];
    }
    if (s > 0)
      out[2 * s - 1] = make_double2(-0.5 * scale * (bk.y - bm.y), 0.5 * scale * (bk.x - bm.x));
    if (s < SEG) {
      double2 C = make_double2(0.5 * (bk.x + bm.x), 0.5 * (bk.y + bm.y));
      if (k == 0) C = cscale(C, 0.5);
      run = cadd(run, C);
      out[2 * s] = run;  // inclusive prefix within the segment (unscaled)
    }
  }
  const double2 off = group_scanE<T>(run, t, f, wsum);
#pragma unroll
  for (int s = 0; s < SEG; ++s) out[2 * s] = cscale(cadd(out[2 * s], off), scale);
  group_sync<T>(f);  // every B read is done: sb may be reused
}

// Pre-processing: v[i] = b_{t + T i} from a loader of a_e (e in [1, M-1]); the
// loader may return garbage for e = 0 and e = M (selected away here).
// dstE_pre_idx: the loader gets (i, mirror) — a_e for e = t + T i, or for
// e = M - t - T i when mirror — so a caller whose addresses are a per-thread base
// plus a compile-time multiple of i can say so. dstE_pre: a loader of e.
template <int P, int E, class Load>
__device__ __forceinline__ void dstE_pre_idx(double2* v, const double* __restrict__ sn,
                                             const EngineTw<P, E>& tw, int t, Load&& load) {
  constexpr int M = FE<P, E>::M, T = FE<P, E>::T, H = M / 2;
  // E = 16: sin(pi (t + T i)/M) = sin(pi t/M) cos(pi i/16) + cos(pi t/M) sin(pi i/16)
  const double st = tw.st, ct = tw.ct;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int e = t + T * i;
    double2 p = load(i, false), q = load(i, true);
    if (i == 0) {
      const bool z = (t == 0);
      p = z ? make_double2(0.0, 0.0) : p;
      q = z ? make_double2(0.0, 0.0) : q;
    }
    double s;
    if constexpr (E == 16) {
      s = fma(st, c32v(i), ct * c32v(i - 8));
    } else {
      s = __ldg(&sn[e <= H ? e : M - e]);
    }
    const double sx = (p.x + q.x) * s, sy = (p.y + q.y) * s;
    v[i] = make_double2(fma(0.5, p.x - q.x, sx), fma(0.5, p.y - q.y, sy));
  }
}

template <int P, int E, class Load>
__device__ __forceinline__ void dstE_pre(double2* v, const double* __restrict__ sn,
                                         const EngineTw<P, E>& tw, int t, Load&& load) {
  constexpr int M = FE<P, E>::M, T = FE<P, E>::T;
  dstE_pre_idx<P, E>(v, sn, tw, t, [&](int i, bool mirror) -> double2 {
    const int e = t + T * i;
    return load(mirror ? M - e : e);
  });
}

}  // namespace hfb
