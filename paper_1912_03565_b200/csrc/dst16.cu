// DST-I along contiguous lines with the register-resident engine (fft16.cuh),
// plus the two y-pass variants with the per-mode Thomas sweep fused in.
//
// Persistent CTAs, each holding NF transform groups. A batch is one plane's
// row group: NF line pairs (2NF lines; pair k = rows (2k, 2k+1), never
// straddling a plane). Input rows are prefetched one batch ahead into shared
// memory with 1D TMA bulk copies (cp.async.bulk + mbarrier, double-buffered),
// so the HBM latency of batch i+1 overlaps the FFT of batch i. Rows need not
// be 16-byte aligned: the copy starts at the aligned address below the row
// and the consumer skips the leading element; a copy that would read past
// the end of the source array is shortened and thread 0 patches the last
// element. Thread 0 resolves every row's addresses per batch into shared
// memory, so the transform threads do no index division.
//
// Modes (MODE template parameter):
//   kRow  : out[plane][row][pos]  — ROW output (the x-iDST writes U)
//   kTran : out[plane][pos][row]  — lines become columns (the x-DST writes
//           the y-pass lines)
//   kYFwd : y-DST of the lines (plane, n, .) followed by the forward Thomas
//           elimination of the modes (n, m = pos) — carry x'_{l-1}, cp_{l-1}
//           from the previous plane; writes x' (in place of the input rows)
//           and cp. One CTA owns a row group for ALL planes, ascending, so the
//           carry is always its own earlier write (tridiag.py:153-165).
//   kYBwd : back substitution W_l = x'_l - cp_l W_{l+1} on the staged x' rows
//           (planes descending, carry W in a per-mode buffer;
//           tridiag.py:166-167), then the inverse y-DST with kTran output.
#include <algorithm>

#include "fft16.cuh"
#include "tma.cuh"

namespace hfb {

enum { kRow = 0, kTran = 1, kYFwd = 2, kYBwd = 3 };  // Dst16Call::mode

struct Fft16 {
  int M, p, T;                     // length, log2, threads per group
  const double2* __restrict__ tw;  // tw[k] = exp(-2 pi i k/M)
  const double* __restrict__ sn;   // sin(pi j/M), j <= M/2
  double scale;                    // sqrt(2/M)
};

struct StreamArgs {
  const double* src;
  double* dst;
  const double* src_end;  // one past the last readable element of src
  int z0, nz;             // first plane, plane count
  int nrow, ppp, G;       // lines per plane, pairs per plane, row groups per plane
  long long in_ld, in_ps, out_ld, out_ps;
  int N, NF, logW;        // line length, groups per CTA, log2(2 NF)
  int rowslot;   // doubles per staged input row (even, >= N + 4)
  int gbuf;      // doubles per group buffer per stage
  int stage_ld;  // output staging row stride (odd, >= N)
  // fused Thomas (kYFwd / kYBwd); rows are x-modes n, positions y-modes m
  double* cp;                       // same layout as the x' rows
  double* wc;                       // kYBwd carry W_{l+1}: one plane, [row * in_ld + pos]
  const double* __restrict__ coef;  // [l][k] (4a, 2b, 2c, d)
  const double* __restrict__ cx;    // cos(pi n/(n_x+1))
  const double* __restrict__ cy;    // cos(pi m/(n_y+1))
  double thr;
  unsigned long long* err;
  int nz_total;                     // levels of the full system (carry ends)
};

constexpr int kMaxRows = 16;  // 2 * NF

struct BatchMeta {
  long long plane[2];
  int row[2][kMaxRows];    // row index within the plane, -1 if absent
  int delta[2][kMaxRows];  // staged-row offset (doubles) of element 0
};

// it-th batch of this CTA -> (plane, row group); false when done.
template <int MODE>
__device__ __forceinline__ bool batch_of(const StreamArgs& a, long long it, long long& plane,
                                         int& g) {
  if (MODE == kYFwd || MODE == kYBwd) {
    const long long gi = it / a.nz;
    const int lp = (int)(it - gi * a.nz);
    const long long gg = blockIdx.x + gi * gridDim.x;
    if (gg >= a.G) return false;
    g = (int)gg;
    plane = a.z0 + (MODE == kYFwd ? lp : a.nz - 1 - lp);
    return true;
  }
  const long long b = blockIdx.x + it * gridDim.x;
  if (b >= (long long)a.nz * a.G) return false;
  plane = a.z0 + b / a.G;
  g = (int)(b % a.G);
  return true;
}

__device__ __forceinline__ double eig(const double* __restrict__ co, double cxv, double cyv) {
  // co = (4a, 2b, 2c, d): lambda = 4a cx cy + 2b cx + 2c cy + d
  return fma(co[0] * cxv + co[2], cyv, fma(co[1], cxv, co[3]));
}

template <int P, int MODE>
__global__ void __launch_bounds__(128, 3) dst16_stream_kernel(StreamArgs a, Fft16 c) {
  extern __shared__ __align__(16) double sm[];
  __shared__ BatchMeta meta;
  constexpr int T = F16<P>::T;
  constexpr bool TRAN = (MODE == kTran || MODE == kYBwd);
  const int f = threadIdx.x / T, t = threadIdx.x - f * T;
  double2* wsum = reinterpret_cast<double2*>(sm + 2LL * a.NF * a.gbuf);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsum + (blockDim.x / 32 + 1));
  auto gbuf = [&](int s, int g) { return sm + ((long long)s * a.NF + g) * a.gbuf; };

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // thread 0: resolve the rows of batch `it` and start their bulk copies into
  // stage s (staged row r at gbuf(s, r/2) + (r&1)*rowslot + 2, 16-B aligned)
  auto issue = [&](long long it, int s) {
    long long plane;
    int g;
    batch_of<MODE>(a, it, plane, g);
    meta.plane[s] = plane;
    uint32_t total = 0;
    const int rows = 2 * a.NF;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) mbar_arrive_expect_tx(&bar[s], total);
#pragma unroll 1
      for (int r = 0; r < rows; ++r) {
        const int k = g * a.NF + (r >> 1);
        const int row = 2 * k + (r & 1);
        if (k >= a.ppp || row >= a.nrow) {
          if (pass == 0) {
            meta.row[s][r] = -1;
            meta.delta[s][r] = 2;
          }
          continue;
        }
        const double* A = a.src + plane * a.in_ps + (long long)row * a.in_ld;
        const double* A16 =
            reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(A) & ~uintptr_t(15));
        const int d = (int)(A - A16);
        uint32_t S = (uint32_t)((8 * (a.N + d) + 15) & ~15);
        const bool cut = A16 + S / 8 > a.src_end;
        if (cut) S -= 16;
        double* dstrow = gbuf(s, r >> 1) + (r & 1) * a.rowslot + 2;
        if (pass == 0) {
          total += S;
          meta.row[s][r] = row;
          meta.delta[s][r] = 2 + d;
          if (cut) dstrow[d + a.N - 1] = __ldg(A + a.N - 1);  // not covered by the copy
        } else {
          bulk_g2s(dstrow, A16, S, &bar[s]);
        }
      }
    }
  };

  long long it = 0;
  int s = 0;
  uint32_t phase0 = 0, phase1 = 0;
  {
    long long pl;
    int g;
    if (threadIdx.x == 0 && batch_of<MODE>(a, 0, pl, g)) issue(0, 0);
  }
  for (;; ++it) {
    long long plane;
    int g;
    if (!batch_of<MODE>(a, it, plane, g)) break;
    {
      long long pl2;
      int g2;
      if (threadIdx.x == 0 && batch_of<MODE>(a, it + 1, pl2, g2)) {
        fence_proxy_async_smem();
        issue(it + 1, s ^ 1);
      }
    }
    mbar_wait(&bar[s], s == 0 ? phase0 : phase1);
    if (s == 0) phase0 ^= 1; else phase1 ^= 1;

    double* gb = gbuf(s, f);
    const int row0 = meta.row[s][2 * f], row1 = meta.row[s][2 * f + 1];
    const bool v0 = row0 >= 0, v1 = row1 >= 0;
    double* r0 = gb + meta.delta[s][2 * f] - 1;  // a_e at r0[e]
    double* r1 = gb + a.rowslot + meta.delta[s][2 * f + 1] - 1;

    if constexpr (MODE == kYBwd) {
      // W_l = x'_l - cp_l W_{l+1} on the staged rows; carry through a.wc
      const int lvl = (int)plane;
      const bool top = (lvl == a.nz_total - 1);
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int row = q ? row1 : row0;
        if (row < 0) continue;
        double* rr = q ? r1 : r0;
        const double* cpr = a.cp + plane * a.in_ps + (long long)row * a.in_ld;
        double* wcr = a.wc + (long long)row * a.in_ld;
        constexpr int NPOS = F16<P>::M - 1;
        constexpr int J = (NPOS + T - 1) / T;
        double cv[J], wv[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int p = t + T * j;
          cv[j] = (!top && p < NPOS) ? __ldg(cpr + p) : 0.0;
          wv[j] = (!top && p < NPOS) ? wcr[p] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int p = t + T * j;
          if (p >= NPOS) continue;
          const double w = fma(-cv[j], wv[j], rr[p + 1]);
          rr[p + 1] = w;
          wcr[p] = w;
        }
      }
      group_sync<T>(f);
    }

    double2 v[16];
    dst16_pre<P>(v, c.sn, t, [&](int e) -> double2 {
      return make_double2(v0 ? r0[e] : 0.0, v1 ? r1[e] : 0.0);
    });
    group_sync<T>(f);  // staged rows consumed: the group buffer becomes FFT scratch
    double2* sb = reinterpret_cast<double2*>(gb);
    fft16_forward<P>(v, sb, c.tw, t, f);
    double2 ev[8], od[8];
    dst16_post<P>(v, sb, wsum, c.scale, t, f, ev, od);
    group_sync<T>(f);
    double* q0 = gb;
    double* q1 = gb + a.stage_ld;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = t + T * i;
      if (k >= 1) {
        q0[2 * k - 1] = ev[i].x;
        q1[2 * k - 1] = ev[i].y;
      }
      q0[2 * k] = od[i].x;
      q1[2 * k] = od[i].y;
    }
    if constexpr (MODE == kRow) {
      group_sync<T>(f);
      const long long b0 = plane * a.out_ps + (long long)row0 * a.out_ld;
      const long long b1 = plane * a.out_ps + (long long)row1 * a.out_ld;
      for (int p = t; p < a.N; p += T) {
        if (v0) a.dst[b0 + p] = q0[p];
        if (v1) a.dst[b1 + p] = q1[p];
      }
    } else if constexpr (MODE == kYFwd) {
      // forward elimination of modes (n = row, m = p) at level l = plane
      group_sync<T>(f);
      const int lvl = (int)plane;
      const double* co = a.coef + (long long)lvl * 12;
      const bool first = (lvl == 0), last = (lvl == a.nz_total - 1);
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int row = q ? row1 : row0;
        if (row < 0) continue;
        const double* qq = q ? q1 : q0;
        const double cxv = __ldg(a.cx + row);
        const long long o = plane * a.out_ps + (long long)row * a.out_ld;
        double* xo = a.dst + o;
        double* co_out = a.cp + o;
        const double* xprev = xo - a.out_ps;
        const double* cprev = co_out - a.out_ps;
        // positions p = t + T j: the carry loads of all j are issued together
        constexpr int NPOS = F16<P>::M - 1;
        constexpr int J = (NPOS + T - 1) / T;
        double xc[J], cc[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int p = t + T * j;
          xc[j] = (!first && p < NPOS) ? xprev[p] : 0.0;
          cc[j] = (!first && p < NPOS) ? cprev[p] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int p = t + T * j;
          if (p >= NPOS) continue;
          const double cyv = __ldg(a.cy + p);
          const double lo = eig(co, cxv, cyv), di = eig(co + 4, cxv, cyv);
          const double den = fma(-lo, cc[j], di);
          const double rhs = fma(-lo, xc[j], qq[p]);
          if (fabs(den) < a.thr) {
            const unsigned long long key =
                ((unsigned long long)lvl * (unsigned long long)NPOS + (unsigned long long)p) *
                    (unsigned long long)a.nrow +
                (unsigned long long)row;
            atomicMin(a.err, key);
          }
          const double rinv = 1.0 / den;
          xo[p] = rhs * rinv;
          if (!last) co_out[p] = eig(co + 8, cxv, cyv) * rinv;
        }
      }
    } else {
      __syncthreads();
      const int W = 2 * a.NF;
      const int total = a.N * W;
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int pos = e >> a.logW, r = e & (W - 1);
        const int row = meta.row[s][r];
        if (row < 0) continue;
        a.dst[plane * a.out_ps + (long long)pos * a.out_ld + row] =
            gbuf(s, r >> 1)[(r & 1) * a.stage_ld + pos];
      }
    }
    __syncthreads();  // stage s is free for the prefetch issued next iteration
    s ^= 1;
  }
}

bool dst16_ok(int M) { return M >= 16 && M <= 4096 && (M & (M - 1)) == 0; }

template <int P, int MODE>
static int launch_stream(const StreamArgs& a, const Fft16& c, int threads, size_t sm,
                         cudaStream_t st) {
  HFB_CUDA(cudaFuncSetAttribute(dst16_stream_kernel<P, MODE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dst16_stream_kernel<P, MODE>,
                                                         threads, sm));
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (MODE == kYFwd || MODE == kYBwd) ? a.G : (long long)a.nz * a.G;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  dst16_stream_kernel<P, MODE><<<(unsigned)blocks, threads, sm, st>>>(a, c);
  return HFB_OK;
}

int launch_dst16_mode(const Dst16Call& k, cudaStream_t st) {
  if (k.nz <= 0 || k.nrow <= 0) return HFB_OK;
  Fft16 c;
  c.M = k.M;
  c.p = 0;
  while ((1 << c.p) < k.M) ++c.p;
  c.T = k.M / 16;
  c.tw = k.tw;
  c.sn = k.sn;
  c.scale = k.scale;
  StreamArgs a;
  a.src = k.src;
  a.src_end = k.src_end;
  a.dst = k.dst;
  a.z0 = k.z0;
  a.nz = k.nz;
  a.nrow = k.nrow;
  a.ppp = (k.nrow + 1) / 2;
  a.in_ld = k.in_ld;
  a.in_ps = k.in_ps;
  a.out_ld = k.out_ld;
  a.out_ps = k.out_ps;
  a.N = k.M - 1;
  a.NF = std::max(1, std::min(128 / c.T, kMaxRows / 2));  // <= 128 threads
  // fused modes: each CTA carries one row group through every plane, so use
  // the smallest groups (most independent chains)
  if (k.mode == kYFwd || k.mode == kYBwd) a.NF = std::max(1, std::min(a.NF, 32 / c.T));
  a.G = (a.ppp + a.NF - 1) / a.NF;
  a.logW = 0;
  while ((1 << a.logW) < 2 * a.NF) ++a.logW;
  a.rowslot = ((a.N + 4) + 1) & ~1;
  a.stage_ld = (a.N % 2 == 1) ? a.N + 2 : a.N + 1;
  a.gbuf = std::max({2 * a.rowslot, 2 * (pad16(k.M) + 1), 2 * a.stage_ld});  // doubles
  a.gbuf = (a.gbuf + 1) & ~1;
  a.cp = k.cp;
  a.wc = k.wc;
  a.coef = k.coef;
  a.cx = k.cx;
  a.cy = k.cy;
  a.thr = k.thr;
  a.err = k.err;
  a.nz_total = k.nz_total;
  const int threads = a.NF * c.T;
  const size_t sm = (size_t)2 * a.NF * a.gbuf * sizeof(double) +
                    (threads / 32 + 1) * sizeof(double2) + 2 * sizeof(uint64_t);
  int rc = HFB_OK;
  switch (c.p) {
#define HFB_P(PP)                                                                       \
  case PP:                                                                              \
    switch (k.mode) {                                                                   \
      case kRow: rc = launch_stream<PP, kRow>(a, c, threads, sm, st); break;            \
      case kTran: rc = launch_stream<PP, kTran>(a, c, threads, sm, st); break;          \
      case kYFwd: rc = launch_stream<PP, kYFwd>(a, c, threads, sm, st); break;          \
      case kYBwd: rc = launch_stream<PP, kYBwd>(a, c, threads, sm, st); break;          \
      default: return HFB_ERR_ARGUMENT;                                                 \
    }                                                                                   \
    break;
    HFB_P(4) HFB_P(5) HFB_P(6) HFB_P(7) HFB_P(8) HFB_P(9) HFB_P(10) HFB_P(11) HFB_P(12)
#undef HFB_P
    default: return HFB_ERR_ARGUMENT;
  }
  if (rc) return rc;
  HFB_LAUNCHED();
  return HFB_OK;
}

int launch_dst16(const double2* tw, const double* sn, double scale, int M, const double* src,
                 const double* src_end, double* dst, int z0, int nz, int nrow, long long in_ld,
                 long long in_ps, long long out_ld, long long out_ps, bool tran,
                 cudaStream_t st) {
  Dst16Call k = {};
  k.mode = tran ? kTran : kRow;
  k.tw = tw;
  k.sn = sn;
  k.scale = scale;
  k.M = M;
  k.src = src;
  k.src_end = src_end;
  k.dst = dst;
  k.z0 = z0;
  k.nz = nz;
  k.nrow = nrow;
  k.in_ld = in_ld;
  k.in_ps = in_ps;
  k.out_ld = out_ld;
  k.out_ps = out_ps;
  return launch_dst16_mode(k, st);
}

}  // namespace hfb
