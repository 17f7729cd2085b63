// DST-I along contiguous lines with the register-resident engine (fft16.cuh).
//
// Persistent CTAs, each holding NF transform groups. A batch is NF line pairs
// (2NF lines); line pair k of a plane = rows (2k, 2k+1), never straddling a
// plane. Input rows are prefetched one batch ahead into shared memory with
// 1D TMA bulk copies (cp.async.bulk + mbarrier, double-buffered), so the HBM
// latency of batch i+1 overlaps the FFT of batch i. Rows need not be 16-byte
// aligned: the copy starts at the aligned address below the row and the
// consumer skips the leading element; a copy that would read past the end of
// the source array is shortened and thread 0 patches the last element.
// Thread 0 also resolves every row's input/output addresses per batch into
// shared memory, so the transform threads do no index division.
//
// Output, staged through shared memory:
//   ROW  : out[plane][row][pos] — each group stores its own two rows;
//   TRAN : out[plane][pos][row] — lines become columns; a warp stores 2NF
//          consecutive rows of 32/(2NF) positions.
#include <algorithm>

#include "fft16.cuh"
#include "tma.cuh"

namespace hfb {

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
  int z0, nrow, ppp;      // first plane, lines per plane, pairs per plane
  long long npairs, nbatch;
  long long in_ld, in_ps, out_ld, out_ps;
  int N, NF, logW;        // line length, groups per CTA, log2(2 NF)
  int rowslot;   // doubles per staged input row (even, >= N + 4)
  int gbuf;      // doubles per group buffer per stage
  int stage_ld;  // output staging row stride (odd, >= N)
};

constexpr int kMaxRows = 16;  // 2 * NF

struct BatchMeta {
  long long out[2][kMaxRows];  // output base offset of each row, -1 if absent
  int delta[2][kMaxRows];      // staged-row offset (doubles) of element 0
};

template <int P, bool TRAN>
__global__ void __launch_bounds__(128, 3) dst16_stream_kernel(StreamArgs a, Fft16 c) {
  extern __shared__ __align__(16) double sm[];
  __shared__ BatchMeta meta;
  constexpr int T = F16<P>::T;
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

  // thread 0: resolve the rows of `batch` and start their bulk copies into
  // stage s (staged row r at gbuf(s, r/2) + (r&1)*rowslot + 2, 16-B aligned)
  auto issue = [&](long long batch, int s) {
    uint32_t total = 0;
    const int rows = 2 * a.NF;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) mbar_arrive_expect_tx(&bar[s], total);
#pragma unroll 1
      for (int r = 0; r < rows; ++r) {
        const long long pr = batch * a.NF + (r >> 1);
        int row = 0;
        long long plane = 0;
        bool valid = pr < a.npairs;
        if (valid) {
          plane = a.z0 + pr / a.ppp;
          row = 2 * (int)(pr % a.ppp) + (r & 1);
          valid = row < a.nrow;
        }
        if (!valid) {
          if (pass == 0) {
            meta.out[s][r] = -1;
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
          meta.delta[s][r] = 2 + d;
          meta.out[s][r] = TRAN ? plane * a.out_ps + row : plane * a.out_ps + row * a.out_ld;
          if (cut) dstrow[d + a.N - 1] = __ldg(A + a.N - 1);  // not covered by the copy
        } else {
          bulk_g2s(dstrow, A16, S, &bar[s]);
        }
      }
    }
  };

  long long batch = blockIdx.x;
  int s = 0;
  uint32_t phase0 = 0, phase1 = 0;
  if (threadIdx.x == 0 && batch < a.nbatch) issue(batch, 0);
  for (; batch < a.nbatch; batch += gridDim.x) {
    const long long next = batch + gridDim.x;
    if (threadIdx.x == 0 && next < a.nbatch) {
      fence_proxy_async_smem();
      issue(next, s ^ 1);
    }
    mbar_wait(&bar[s], s == 0 ? phase0 : phase1);
    if (s == 0) phase0 ^= 1; else phase1 ^= 1;

    double* gb = gbuf(s, f);
    const double* r0 = gb + meta.delta[s][2 * f] - 1;            // a_e at r0[e]
    const double* r1 = gb + a.rowslot + meta.delta[s][2 * f + 1] - 1;
    const bool v0 = meta.out[s][2 * f] >= 0, v1 = meta.out[s][2 * f + 1] >= 0;
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
    if (!TRAN) {
      group_sync<T>(f);
      const long long b0 = meta.out[s][2 * f], b1 = meta.out[s][2 * f + 1];
      for (int p = t; p < a.N; p += T) {
        if (b0 >= 0) a.dst[b0 + p] = q0[p];
        if (b1 >= 0) a.dst[b1 + p] = q1[p];
      }
    } else {
      __syncthreads();
      const int W = 2 * a.NF;
      const int total = a.N * W;
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int pos = e >> a.logW, r = e & (W - 1);
        const long long base = meta.out[s][r];
        if (base < 0) continue;
        a.dst[base + (long long)pos * a.out_ld] = gbuf(s, r >> 1)[(r & 1) * a.stage_ld + pos];
      }
    }
    __syncthreads();  // stage s is free for the prefetch issued next iteration
    s ^= 1;
  }
}

bool dst16_ok(int M) { return M >= 16 && M <= 4096 && (M & (M - 1)) == 0; }

template <int P, bool TRAN>
static int launch_stream(const StreamArgs& a, const Fft16& c, int threads, size_t sm,
                         cudaStream_t st) {
  HFB_CUDA(cudaFuncSetAttribute(dst16_stream_kernel<P, TRAN>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dst16_stream_kernel<P, TRAN>,
                                                         threads, sm));
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long blocks = std::min<long long>(a.nbatch, (long long)sms * std::max(per_sm, 1));
  dst16_stream_kernel<P, TRAN><<<(unsigned)blocks, threads, sm, st>>>(a, c);
  return HFB_OK;
}

// Lines (plane z0.., nrow lines each, line stride in_ld, plane stride in_ps)
// -> ROW (out_ld line stride) or TRAN (out_ld position stride).
// src_end: one past the last element that may be read from src.
int launch_dst16(const double2* tw, const double* sn, double scale, int M, const double* src,
                 const double* src_end, double* dst, int z0, int nz, int nrow, long long in_ld,
                 long long in_ps, long long out_ld, long long out_ps, bool tran,
                 cudaStream_t st) {
  if (nz <= 0 || nrow <= 0) return HFB_OK;
  Fft16 c;
  c.M = M;
  c.p = 0;
  while ((1 << c.p) < M) ++c.p;
  c.T = M / 16;
  c.tw = tw;
  c.sn = sn;
  c.scale = scale;
  StreamArgs a;
  a.src = src;
  a.src_end = src_end;
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
  a.NF = std::max(1, std::min(128 / c.T, kMaxRows / 2));  // <= 128 threads
  a.logW = 0;
  while ((1 << a.logW) < 2 * a.NF) ++a.logW;
  a.nbatch = (a.npairs + a.NF - 1) / a.NF;
  a.rowslot = ((a.N + 4) + 1) & ~1;
  a.stage_ld = (a.N % 2 == 1) ? a.N + 2 : a.N + 1;
  a.gbuf = std::max({2 * a.rowslot, 2 * (pad16(M) + 1), 2 * a.stage_ld});  // doubles
  a.gbuf = (a.gbuf + 1) & ~1;
  const int threads = a.NF * c.T;
  const size_t sm = (size_t)2 * a.NF * a.gbuf * sizeof(double) +
                    (threads / 32 + 1) * sizeof(double2) + 2 * sizeof(uint64_t);
  int rc = HFB_OK;
  switch (c.p) {
#define HFB_P(PP)                                                              \
  case PP:                                                                     \
    rc = tran ? launch_stream<PP, true>(a, c, threads, sm, st)                 \
              : launch_stream<PP, false>(a, c, threads, sm, st);               \
    break;
    HFB_P(4) HFB_P(5) HFB_P(6) HFB_P(7) HFB_P(8) HFB_P(9) HFB_P(10) HFB_P(11) HFB_P(12)
#undef HFB_P
    default: return HFB_ERR_ARGUMENT;
  }
  if (rc) return rc;
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb
