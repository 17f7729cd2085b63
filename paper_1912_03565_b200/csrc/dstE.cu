// DST-I along contiguous lines with the register-resident engine (fftE.cuh).
//
// Persistent CTAs, each holding NF transform groups (one warp per group for
// M = 1024). A batch is one plane's row group: NF line pairs (2NF lines; pair
// k = rows (2k, 2k+1), never straddling a plane). Input rows are prefetched
// one batch ahead into shared memory with 1D TMA bulk copies (cp.async.bulk +
// mbarrier, double-buffered), so the HBM latency of batch i+1 overlaps the
// transform of batch i. Rows need not be 16-byte aligned: the copy starts at
// the aligned address below the row and the consumer skips the leading
// element; a copy that would read past the end of the source array is
// shortened and thread 0 patches the last element. Thread 0 resolves every
// row's addresses per batch into shared memory.
//
// Output, staged through shared memory (rows padded one slot per 32):
//   ROW  : out[plane][row][pos] — each group stores its own two rows;
//   TRAN : out[plane][pos][row] — lines become columns; a warp stores 2NF
//          consecutive rows of 32/(2NF) positions.
#include <algorithm>

#include "fftE.cuh"
#include "tma.cuh"

namespace hfb {

enum { kRow = 0, kTran = 1 };  // Dst16Call::mode

struct FftArgs {
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
  int stage_ld;  // output staging row stride (odd, > pad32(N + 1))
};

constexpr int kMaxRows = 16;  // 2 * NF

struct BatchMeta {
  long long plane[2];
  int row[2][kMaxRows];    // row index within the plane, -1 if absent
  int delta[2][kMaxRows];  // staged-row offset (doubles) of element 0
};

__device__ __forceinline__ bool batch_of(const StreamArgs& a, long long it, long long& plane,
                                         int& g) {
  const long long b = blockIdx.x + it * gridDim.x;
  if (b >= (long long)a.nz * a.G) return false;
  plane = a.z0 + b / a.G;
  g = (int)(b % a.G);
  return true;
}

template <int P, int E, int MODE>
__global__ void __launch_bounds__(128, 3) dstE_stream_kernel(StreamArgs a, FftArgs c) {
  extern __shared__ __align__(16) double sm[];
  __shared__ BatchMeta meta;
  constexpr int T = FE<P, E>::T, SEG = FE<P, E>::SEG;
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
    batch_of(a, it, plane, g);
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

  int s = 0;
  uint32_t phase0 = 0, phase1 = 0;
  {
    long long pl;
    int g;
    if (threadIdx.x == 0 && batch_of(a, 0, pl, g)) issue(0, 0);
  }
  for (long long it = 0;; ++it) {
    long long plane;
    int g;
    if (!batch_of(a, it, plane, g)) break;
    {
      long long pl2;
      int g2;
      if (threadIdx.x == 0 && batch_of(a, it + 1, pl2, g2)) {
        fence_proxy_async_smem();
        issue(it + 1, s ^ 1);
      }
    }
    mbar_wait(&bar[s], s == 0 ? phase0 : phase1);
    if (s == 0) phase0 ^= 1; else phase1 ^= 1;

    double* gb = gbuf(s, f);
    const int row0 = meta.row[s][2 * f], row1 = meta.row[s][2 * f + 1];
    const bool v0 = row0 >= 0, v1 = row1 >= 0;
    const double* r0 = gb + meta.delta[s][2 * f] - 1;  // a_e at r0[e]
    const double* r1 = gb + a.rowslot + meta.delta[s][2 * f + 1] - 1;

    double2 v[E];
    dstE_pre<P, E>(v, c.sn, t, [&](int e) -> double2 {
      return make_double2(v0 ? r0[e] : 0.0, v1 ? r1[e] : 0.0);
    });
    group_sync<T>(f);  // staged rows consumed: the group buffer becomes FFT scratch
    double2* sb = reinterpret_cast<double2*>(gb);
    fftE_forward<P, E>(v, sb, c.tw, t, f);
    double2 out[2 * SEG];
    dstE_post<P, E>(v, sb, wsum, c.scale, t, f, out);
    // stage: position p of row q at gb[q * stage_ld + pad32(p + 1)]
    double* q0 = gb;
    double* q1 = gb + a.stage_ld;
#pragma unroll
    for (int j = 0; j < 2 * SEG; ++j) {
      const int idx = pad32(2 * SEG * t + j);  // position 2 SEG t + j - 1, shifted by one
      if (t > 0 || j > 0) {
        q0[idx] = out[j].x;
        q1[idx] = out[j].y;
      }
    }
    if constexpr (MODE == kRow) {
      group_sync<T>(f);
      const long long b0 = plane * a.out_ps + (long long)row0 * a.out_ld;
      const long long b1 = plane * a.out_ps + (long long)row1 * a.out_ld;
      for (int p = t; p < a.N; p += T) {
        if (v0) a.dst[b0 + p] = q0[pad32(p + 1)];
        if (v1) a.dst[b1 + p] = q1[pad32(p + 1)];
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
            gbuf(s, r >> 1)[(r & 1) * a.stage_ld + pad32(pos + 1)];
      }
    }
    __syncthreads();  // stage s is free for the prefetch issued next iteration
    s ^= 1;
  }
}

bool dst16_ok(int M) { return M >= 16 && M <= 4096 && (M & (M - 1)) == 0; }

template <int P, int E, int MODE>
static int launch_stream(const StreamArgs& a, const FftArgs& c, int threads, size_t sm,
                         cudaStream_t st) {
  auto kern = dstE_stream_kernel<P, E, MODE>;
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, sm));
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nz * a.G;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  kern<<<(unsigned)blocks, threads, sm, st>>>(a, c);
  return HFB_OK;
}

// tuning knobs (hfb_set_tuning): engine width E for M >= 32 and groups per CTA
static int g_tune_E = 16;
static int g_tune_NF = 0;

template <int P, int E>
static int launch_pe(const Dst16Call& k, StreamArgs a, const FftArgs& c, cudaStream_t st) {
  constexpr int T = FE<P, E>::T;
  a.NF = std::max(1, std::min(128 / T, kMaxRows / 2));  // <= 128 threads per CTA
  if (g_tune_NF > 0) a.NF = std::max(1, std::min(g_tune_NF, std::min(128 / T, kMaxRows / 2)));
  a.G = (a.ppp + a.NF - 1) / a.NF;
  a.logW = 0;
  while ((1 << a.logW) < 2 * a.NF) ++a.logW;
  a.rowslot = ((a.N + 4) + 1) & ~1;
  a.stage_ld = pad32(a.N + 1) + 1;
  if (a.stage_ld % 2 == 0) ++a.stage_ld;
  a.gbuf = std::max({2 * a.rowslot, 2 * FE<P, E>::BUF, 2 * a.stage_ld});  // doubles
  a.gbuf = (a.gbuf + 1) & ~1;
  const int threads = a.NF * T;
  const size_t sm = (size_t)2 * a.NF * a.gbuf * sizeof(double) +
                    (threads / 32 + 1) * sizeof(double2) + 2 * sizeof(uint64_t);
  if (k.mode == kTran) return launch_stream<P, E, kTran>(a, c, threads, sm, st);
  return launch_stream<P, E, kRow>(a, c, threads, sm, st);
}

template <int P>
static int launch_p(const Dst16Call& k, StreamArgs a, const FftArgs& c, cudaStream_t st) {
  if constexpr (P >= 5) {
    if (g_tune_E == 32) return launch_pe<P, 32>(k, a, c, st);
  }
  return launch_pe<P, 16>(k, a, c, st);
}

void set_tuning(int key, int value) {
  if (key == 0) g_tune_E = (value == 32) ? 32 : 16;
  if (key == 1) g_tune_NF = value;
}

int launch_dst16_mode(const Dst16Call& k, cudaStream_t st) {
  if (k.nz <= 0 || k.nrow <= 0) return HFB_OK;
  if (k.mode != kRow && k.mode != kTran) return HFB_ERR_ARGUMENT;
  int p = 0;
  while ((1 << p) < k.M) ++p;
  FftArgs c;
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
  int rc = HFB_OK;
  switch (p) {
#define HFB_P(PP) \
  case PP: rc = launch_p<PP>(k, a, c, st); break;
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
