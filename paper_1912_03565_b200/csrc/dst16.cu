// DST-I along contiguous lines with the register-resident engine (fft16.cuh).
//
// Persistent CTAs, each holding NF transform groups. A batch is NF line pairs
// (2NF lines); line pair k of a plane = rows (2k, 2k+1), never straddling a
// plane. Input rows are prefetched one batch ahead into shared memory with
// 1D TMA bulk copies (cp.async.bulk + mbarrier, double-buffered), so the HBM
// latency of batch i+1 overlaps the FFT of batch i. Rows need not be 16-byte
// aligned: the copy starts at the aligned address below the row and the
// consumer skips the leading element.
//
// Output, staged through shared memory:
//   ROW  : out[plane][row][pos] — each group stores its own two rows,
//          coalesced;
//   TRAN : out[plane][pos][row] — lines become columns; a warp stores 2NF
//          consecutive rows of 32/(2NF) positions.
// The x-pass uses TRAN into a padded scratch (lines of the y-pass); the
// y-pass uses TRAN back into the natural (m, n) order.
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
  int N, NF;
  int rowslot;   // doubles per staged input row (even, >= N + 2)
  int gbuf;      // doubles per group buffer per stage
  int stage_ld;  // output staging row stride (odd, >= N)
};

struct RowRef {
  long long plane;
  int row;
  bool valid;
};

__device__ __forceinline__ RowRef batch_row(const StreamArgs& a, long long batch, int r) {
  RowRef x;
  const long long pr = batch * a.NF + (r >> 1);
  x.valid = pr < a.npairs;
  x.plane = x.valid ? a.z0 + pr / a.ppp : 0;
  x.row = x.valid ? 2 * (int)(pr % a.ppp) + (r & 1) : 0;
  x.valid = x.valid && x.row < a.nrow;
  return x;
}

template <int P, bool TRAN>
__global__ void __launch_bounds__(128, 3) dst16_stream_kernel(StreamArgs a, Fft16 c) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_delta[2][16];
  __shared__ int s_tail[2][16];
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

  // thread 0: start the bulk copies of `batch` into stage s. Row r is copied
  // from the 16-byte aligned address at or below its start; `delta` is the
  // number of leading doubles to skip; a row whose rounded-up copy would read
  // past src_end drops its last 16 bytes and the consumer loads the tail.
  auto row_copy = [&](long long batch, int r, const double*& A16, uint32_t& S, int& d,
                      int& tail) {
    const RowRef x = batch_row(a, batch, r);
    S = 0;
    d = 0;
    tail = 0;
    if (!x.valid) return;
    const double* A = a.src + x.plane * a.in_ps + (long long)x.row * a.in_ld;
    A16 = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(A) & ~uintptr_t(15));
    d = (int)(A - A16);
    S = (uint32_t)((8 * (a.N + d) + 15) & ~15);
    if (A16 + S / 8 > a.src_end) {
      S -= 16;
      tail = 1;
    }
  };
  auto issue = [&](long long batch, int s) {
    uint32_t total = 0;
#pragma unroll 1
    for (int r = 0; r < 2 * a.NF; ++r) {
      const double* A16;
      uint32_t S;
      int d, tail;
      row_copy(batch, r, A16, S, d, tail);
      total += S;
      s_delta[s][r] = d;
      s_tail[s][r] = tail;
    }
    mbar_arrive_expect_tx(&bar[s], total);
#pragma unroll 1
    for (int r = 0; r < 2 * a.NF; ++r) {
      const double* A16;
      uint32_t S;
      int d, tail;
      row_copy(batch, r, A16, S, d, tail);
      if (S) bulk_g2s(gbuf(s, r >> 1) + (r & 1) * a.rowslot, A16, S, &bar[s]);
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
    const RowRef x0 = batch_row(a, batch, 2 * f), x1 = batch_row(a, batch, 2 * f + 1);
    const double* r0 = gb + s_delta[s][2 * f];
    const double* r1 = gb + a.rowslot + s_delta[s][2 * f + 1];
    const bool t0 = s_tail[s][2 * f], t1 = s_tail[s][2 * f + 1];
    const int last = a.N - 1;
    const double* g0 = a.src + x0.plane * a.in_ps + (long long)x0.row * a.in_ld;
    const double* g1 = a.src + x1.plane * a.in_ps + (long long)x1.row * a.in_ld;
    double2 v[16];
    dst16_pre<P>(v, c.sn, t, [&](int e) -> double2 {
      const int p = e - 1;
      double xr = 0.0, xi = 0.0;
      if (x0.valid) xr = (t0 && p == last) ? __ldg(g0 + p) : r0[p];
      if (x1.valid) xi = (t1 && p == last) ? __ldg(g1 + p) : r1[p];
      return make_double2(xr, xi);
    });
    __syncthreads();  // staged rows consumed: the group buffer becomes FFT scratch
    double2* sb = reinterpret_cast<double2*>(gb);
    fft16_forward<P>(v, sb, c.tw, t);
    double2 ev[8], od[8];
    dst16_post<P>(v, sb, wsum, c.scale, t, ev, od);
    __syncthreads();
    // stage rows [2f, 2f+1] x positions
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
    __syncthreads();
    if (!TRAN) {
      double* o0 = a.dst + x0.plane * a.out_ps + (long long)x0.row * a.out_ld;
      double* o1 = a.dst + x1.plane * a.out_ps + (long long)x1.row * a.out_ld;
      for (int p = t; p < a.N; p += T) {
        if (x0.valid) o0[p] = q0[p];
        if (x1.valid) o1[p] = q1[p];
      }
    } else {
      const int W = 2 * a.NF;
      const int total = a.N * W;
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int pos = e / W, r = e - pos * W;
        const RowRef x = batch_row(a, batch, r);
        if (!x.valid) continue;
        a.dst[x.plane * a.out_ps + (long long)pos * a.out_ld + x.row] =
            gbuf(s, r >> 1)[(r & 1) * a.stage_ld + pos];
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
  a.NF = std::max(1, std::min(128 / c.T, 8));  // <= 128 threads, <= 16 rows per batch
  a.nbatch = (a.npairs + a.NF - 1) / a.NF;
  a.rowslot = ((a.N + 2) + 1) & ~1;
  a.stage_ld = (a.N % 2 == 1) ? a.N + 2 : a.N + 1;
  a.gbuf = std::max({2 * a.rowslot, 2 * (pad16(M) + 1), 2 * a.stage_ld});  // doubles
  a.gbuf = (a.gbuf + 1) & ~1;
  const int threads = a.NF * c.T;
  const size_t sm = (size_t)2 * a.NF * a.gbuf * sizeof(double) +
                    (threads / 32 + 1) * sizeof(double2) + 2 * sizeof(uint64_t);
  int per_sm = 1;
  int rc = HFB_OK;
  switch (c.p) {
#define HFB_P(PP)                                                                 \
  case PP:                                                                        \
    rc = tran ? launch_stream<PP, true>(a, c, threads, sm, st)                    \
              : launch_stream<PP, false>(a, c, threads, sm, st);                  \
    break;
    HFB_P(4) HFB_P(5) HFB_P(6) HFB_P(7) HFB_P(8) HFB_P(9) HFB_P(10) HFB_P(11) HFB_P(12)
#undef HFB_P
    default: return HFB_ERR_ARGUMENT;
  }
  (void)per_sm;
  if (rc) return rc;
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb
