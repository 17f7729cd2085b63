// Transpose-free distributed z-solve ("alternative to
// measure next"): every rank keeps its z-slab of mode rows (kpz, n_x, ld) for
// the whole solve, and the N_x N_y tridiagonal systems are swept ACROSS the
// ranks instead of being gathered onto one rank by an all-to-all.
//
//   forward  on rank p: elimination over levels z0 .. z1-1 needs (x', cp) at
//            level z0 - 1, the last forward level of rank p - 1;
//   backward on rank p: back substitution over z1-1 .. z0 needs W at level z1,
//            the last backward level of rank p + 1.
//
// The carries travel per block of 256 modes (one row segment, as in
// thomas_tma.cu) through peer memory: the kernel stores a finished block's
// carry straight into the neighbour's carry region (NVLink stores to an
// IPC-mapped allocation), fences, and publishes the block with a release
// store of the solve's epoch into the neighbour's flag. The neighbour's CTA for
// that block spins on the flag (acquire) after issuing its first TMA loads, so
// rank p + 1 starts block b as soon as rank p has finished it: a pipeline over
// mode blocks with O(n_x n_y) bytes per boundary instead of two full-volume
// all-to-alls. A flag that never arrives latches an exchange error after a
// timeout instead of hanging the GPU (reported as ExchangeError).
//
// Per block the data moves exactly as in thomas_tma.cu (8-level chunks by 1D
// bulk copies into a 3-stage ring, bulk stores out, cp checkpointed once per
// chunk and recomputed in the back substitution), and the arithmetic is the
// same expression for expression, so the distributed solve equals the one-call
// solve bit for bit.
//
// Carry region of a rank (doubles; A = n_x * ld):
//   [0, A)   x' at level z0 - 1   (written by rank p - 1)
//   [A, 2A)  cp at level z0 - 1   (written by rank p - 1)
//   [2A, 3A) W at level z1        (written by rank p + 1)
//   then uint32 flags: nblk forward (by rank p - 1), nblk backward (by p + 1)
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "hfb_internal.cuh"
#include "tma.cuh"

namespace hfb {

namespace {
constexpr int BM = 256;
constexpr int K = kThomasChunk;
constexpr int SMAX = 6;  // ring stages: 3 at full occupancy, 6 with one or two CTAs per SM

struct CarryArgs {
  double* w;            // local slab: local level l at w + l * ps
  double* cpk;          // local checkpoints: plane q = cp at local level q*K + K - 1
  const double* coef;   // global weights [l][k][(4a, 2b, 2c, d)]
  const double* cx;
  const double* cy;
  int nzl, z0, nz;      // local levels, global level of local level 0, global levels
  int nrows, ncols, nbpr;
  long long ld, ps;
  double thr;
  unsigned long long* err;
  double* mine;         // this rank's carry region
  double* peer;         // the neighbour's (next: forward, previous: backward) or null
  unsigned epoch;
  unsigned long long timeout_ns;
  unsigned* xerr;
  int zinv;  // z-invariant weights: eigenvalues once per block, no weight copies
  const double* pq;  // [n][l][k][(P, Q)] of the real table (hfb_plan::pq)
};

// real weights: the shared P cy + Q order (hfb_internal.cuh), as the one-call sweep
__device__ __forceinline__ double eig_c(const double* co, double cx, double cy, double cxy) {
  (void)cxy;
  return eig_pq(co, cx, cy);
}
// complex weights (re, im parts apiece): thomas_tma_z.cu's order, which the
// complex one-call solve uses
__device__ __forceinline__ double eig_cz(const double* co, double cx, double cy, double cxy) {
  return fma(co[0], cxy, fma(co[1], cx, fma(co[2], cy, co[3])));
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Thread 0: wait until the neighbour published this block for `epoch` (wrap-safe
// compare). Gives up after the timeout, or at once when another CTA already
// did, latching `code` (1: forward carry missing, 2: backward carry missing).
__device__ void wait_block(const unsigned* flag, unsigned epoch, unsigned long long timeout,
                           unsigned* xerr, unsigned code) {
  const unsigned long long t0 = global_ns();
  for (;;) {
    if ((int)(ld_acquire_sys(flag) - epoch) >= 0) return;
    if (*(volatile unsigned*)xerr) return;
    if (global_ns() - t0 > timeout) {
      atomicCAS(xerr, 0u, code);
      return;
    }
    __nanosleep(200);
  }
}

// thread 0: bring local chunk c (levels c*K ..) and its weights into stage s
__device__ __forceinline__ void issue_chunk(const CarryArgs& a, double (*sdat)[K][BM],
                                            double (*scoef)[K * 12], uint64_t* bar,
                                            const double* base, uint32_t rowbytes, int c, int s,
                                            int n) {
  const int l0 = c * K, nl = min(K, a.nzl - l0);
  mbar_arrive_expect_tx(&bar[s], nl * rowbytes + (a.zinv ? 0u : (uint32_t)(nl * 6 * 8)));
  for (int i = 0; i < nl; ++i) bulk_g2s(&sdat[s][i][0], base + (long long)(l0 + i) * a.ps, rowbytes, &bar[s]);
  if (!a.zinv)  // the block's x-mode's (P, Q) pairs of these levels
    bulk_g2s(&scoef[s][0], a.pq + ((long long)n * a.nz + a.z0 + l0) * 6, (uint32_t)(nl * 6 * 8),
             &bar[s]);
}
}  // namespace

// DIR 0: forward elimination (chunks ascending), DIR 1: back substitution
// (chunks descending); one launch per direction and rank. The CTA walks the
// mode blocks cta, cta + ncta, ... (ascending: a block waits only on the same
// block of the neighbour, which that rank's CTA reaches no later).
template <int DIR, int S, bool ZI>
__device__ __forceinline__ void carry_body(const CarryArgs& a, long long cta, long long ncta) {
  extern __shared__ __align__(16) double dyn[];
  double(*sdat)[K][BM] = reinterpret_cast<double(*)[K][BM]>(dyn);
  double(*scoef)[K * 12] = reinterpret_cast<double(*)[K * 12]>(dyn + S * K * BM);
  __shared__ uint64_t bar[S];
  const int tid = threadIdx.x;
  const int nchunk = (a.nzl + K - 1) / K;
  const long long A = (long long)a.nrows * a.ld;
  const long long nblk = (long long)a.nrows * a.nbpr;
  const bool has_prev = a.z0 > 0, has_next = a.z0 + a.nzl < a.nz;
  unsigned* flags_mine = reinterpret_cast<unsigned*>(a.mine + 3 * A) + (DIR ? nblk : 0);
  unsigned* flags_peer =
      a.peer ? reinterpret_cast<unsigned*>(a.peer + 3 * A) + (DIR ? nblk : 0) : nullptr;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase = 0;

  for (long long blk = cta; blk < nblk; blk += ncta) {
    const int n = (int)(blk / a.nbpr);
    const int m0 = (int)(blk % a.nbpr) * BM;
    const int cols = min(BM, a.ncols - m0);
    const uint32_t rowbytes = (uint32_t)(((cols + 1) & ~1) * 8);  // ld is even
    double* base = a.w + (long long)n * a.ld + m0;
    auto chunk_of = [&](int task) { return DIR ? nchunk - 1 - task : task; };
    const bool live = tid < cols;
    const int m = m0 + tid;
    const long long idx = (long long)n * a.ld + m;
    const double cxv = __ldg(a.cx + n);
    const double cyv = live ? __ldg(a.cy + m) : 0.0;
    const double cxy = cxv * cyv;
    double* ck = a.cpk + (long long)n * a.ld + m0 + tid;
    // z-invariant weights (thomas_tma.cu, tuning key 31): the mode's three
    // eigenvalues once per block, the same expressions and bits
    double zl = 0.0, zd = 0.0, zu = 0.0;
    if constexpr (ZI) {
      zl = eig_c(a.coef, cxv, cyv, cxy);
      zd = eig_c(a.coef + 4, cxv, cyv, cxy);
      zu = eig_c(a.coef + 8, cxv, cyv, cxy);
    }
    if (tid == 0) {
      for (int t = 0; t < S - 1 && t < nchunk; ++t)
        issue_chunk(a, sdat, scoef, bar, base, rowbytes, chunk_of(t), t, n);
    }
    // the carry in: forward (x', cp) at z0 - 1, backward W at z1
    double c = 0.0, x = 0.0;
    const bool wait_in = DIR ? has_next : has_prev;
    if (wait_in) {
      if (tid == 0) wait_block(flags_mine + blk, a.epoch, a.timeout_ns, a.xerr, DIR ? 2u : 1u);
      __syncthreads();
      if (live) {
        if (DIR) {
          x = __ldcg(a.mine + 2 * A + idx);
        } else {
          x = __ldcg(a.mine + idx);
          c = __ldcg(a.mine + A + idx);
        }
      }
    }
    // backward: cp at the level below each chunk (checkpoint, or the forward
    // carry-in below local level 0), one chunk ahead
    auto cp_below = [&](int cidx) -> double {
      if (!live) return 0.0;
      if (cidx > 0) return ck[(long long)(cidx - 1) * a.ps];
      return has_prev ? __ldcg(a.mine + A + idx) : 0.0;
    };
    double cbelow = DIR ? cp_below(chunk_of(0)) : 0.0;
    for (int task = 0; task < nchunk; ++task) {
      const int s = task % S;
      if (tid == 0 && task + S - 1 < nchunk) {
        bulk_wait_read<0>();  // stage s' was stored from at task - 1
        fence_proxy_async_smem();
        issue_chunk(a, sdat, scoef, bar, base, rowbytes, chunk_of(task + S - 1),
                       (task + S - 1) % S, n);
      }
      mbar_wait(&bar[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const int cidx = chunk_of(task);
      const int l0 = cidx * K, nl = min(K, a.nzl - l0);
      const double* co = &scoef[s][0];
      if (DIR == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i < nl) {
            const int l = a.z0 + l0 + i;
            const double lo = (ZI ? zl : fma(co[i * 6], cyv, co[i * 6 + 1]));
            const double di = (ZI ? zd : fma(co[i * 6 + 2], cyv, co[i * 6 + 3]));
            const double up = (ZI ? zu : fma(co[i * 6 + 4], cyv, co[i * 6 + 5]));
            const double den = (l == 0) ? di : fma(-lo, c, di);
            if (live && fabs(den) < a.thr) {
              const unsigned long long key =
                  ((unsigned long long)l * (unsigned long long)a.ncols + (unsigned long long)m) *
                      (unsigned long long)a.nrows +
                  (unsigned long long)n;
              atomicMin(a.err, key);
            }
            const double rr = rcp_fast(den);
            x = ((l == 0) ? sdat[s][i][tid] : fma(-lo, x, sdat[s][i][tid])) * rr;
            sdat[s][i][tid] = x;
            if (l < a.nz - 1) {
              c = up * rr;
              if (i == K - 1 && live) ck[(long long)cidx * a.ps] = c;
            }
          }
        }
      } else {
        double cprev = cbelow;
        if (task + 1 < nchunk) cbelow = cp_below(chunk_of(task + 1));
        double cb[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int l = a.z0 + l0 + i;
          if (i < nl && l < a.nz - 1) {
            const double di = (ZI ? zd : fma(co[i * 6 + 2], cyv, co[i * 6 + 3]));
            const double lo = (ZI ? zl : fma(co[i * 6], cyv, co[i * 6 + 1]));
            const double dl = (l == 0) ? di : fma(-lo, cprev, di);
            const double rr = rcp_fast(dl);
            cprev = (ZI ? zu : fma(co[i * 6 + 4], cyv, co[i * 6 + 5])) * rr;
            cb[i] = cprev;
          }
        }
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
          const int l = a.z0 + l0 + i;
          if (i < nl) {
            if (l < a.nz - 1) {
              x = fma(-cb[i], x, sdat[s][i][tid]);
              sdat[s][i][tid] = x;
            } else {
              x = sdat[s][i][tid];  // top of the system: W = x'
            }
          }
        }
      }
      __syncthreads();  // every thread's results for this chunk are in sdat[s]
      if (tid == 0) {
        fence_proxy_async_smem();
        for (int i = 0; i < nl; ++i)
          bulk_s2g(base + (long long)(l0 + i) * a.ps, &sdat[s][i][0], rowbytes);
        bulk_commit();
      }
    }
    // the carry out, published per block
    const bool send = DIR ? has_prev : has_next;
    if (send) {
      if (live) {
        if (DIR) {
          a.peer[2 * A + idx] = x;
        } else {
          a.peer[idx] = x;
          a.peer[A + idx] = c;
        }
      }
      __threadfence_system();
      __syncthreads();
      if (tid == 0) st_release_sys(flags_peer + blk, a.epoch);
    }
    if (tid == 0) bulk_wait<0>();  // stores done before the stages are refilled
    __syncthreads();
  }
}

template <int DIR, int S, bool ZI>
__global__ void __launch_bounds__(BM, 4) thomas_carry_kernel(CarryArgs a) {
  carry_body<DIR, S, ZI>(a, blockIdx.x, gridDim.x);
}

// Verification of the cross-rank protocol on ONE device: every virtual rank's
// sweep in ONE cooperative launch (all CTAs co-resident), CTA group r serving
// rank r. Rank r's CTAs really spin on flags that rank r -/+ 1's CTAs release
// while running concurrently — the live acquire/release path of the
// multi-GPU run, without separate launches waiting on one another.
template <int DIR, int S, bool ZI>
__global__ void __launch_bounds__(BM, 4) thomas_carry_vranks_kernel(const CarryArgs* va, int per) {
  const int r = blockIdx.x / per;
  const CarryArgs a = va[r];
  carry_body<DIR, S, ZI>(a, blockIdx.x - (long long)r * per, per);
}

// ---------------------------------------------------------------------------
// Complex coefficients (complex k(z)) across ranks: the same
// pipeline on two real volumes (re, im) with thomas_tma_z.cu's complex
// arithmetic, expression for expression. Carry region (doubles, A = n_x ld):
//   [0, 2A)  x' re, im at z0 - 1;  [2A, 4A) cp re, im at z0 - 1;
//   [4A, 6A) W re, im at z1;       then nblk forward + nblk backward flags.
namespace {
struct cz2 {
  double r, i;
};
__device__ __forceinline__ cz2 zmul2(cz2 a, cz2 b) {
  return {fma(a.r, b.r, -a.i * b.i), fma(a.r, b.i, a.i * b.r)};
}
__device__ __forceinline__ cz2 zfms2(cz2 a, cz2 b, cz2 c) {  // a - b * c
  return {fma(-b.r, c.r, fma(b.i, c.i, a.r)), fma(-b.r, c.i, fma(-b.i, c.r, a.i))};
}
__device__ __forceinline__ cz2 zrcp2(cz2 d, double& n2) {
  n2 = fma(d.r, d.r, d.i * d.i);
  const double inv = 1.0 / n2;
  return {d.r * inv, -d.i * inv};
}

struct CarryZArgs {
  double* wr;
  double* wi;
  double* cpk;  // chunk q: re at plane 2q, im at 2q + 1
  const double* coefr;
  const double* coefi;
  const double* cx;
  const double* cy;
  int nzl, z0, nz;
  int nrows, ncols, nbpr;
  long long ld, ps;
  double thr2;
  unsigned long long* err;
  double* mine;
  double* peer;
  unsigned epoch;
  unsigned long long timeout_ns;
  unsigned* xerr;
};
}  // namespace

template <int DIR>
__global__ void __launch_bounds__(BM) thomas_carry_z_kernel(CarryZArgs a) {
  constexpr int S = 3;
  extern __shared__ __align__(16) double dyn[];
  double(*sdat)[2][K][BM] = reinterpret_cast<double(*)[2][K][BM]>(dyn);
  double(*scoef)[2][K * 12] = reinterpret_cast<double(*)[2][K * 12]>(dyn + S * 2 * K * BM);
  __shared__ uint64_t bar[S];
  const int tid = threadIdx.x;
  const int nchunk = (a.nzl + K - 1) / K;
  const long long A = (long long)a.nrows * a.ld;
  const long long nblk = (long long)a.nrows * a.nbpr;
  const bool has_prev = a.z0 > 0, has_next = a.z0 + a.nzl < a.nz;
  unsigned* flags_mine = reinterpret_cast<unsigned*>(a.mine + 6 * A) + (DIR ? nblk : 0);
  unsigned* flags_peer =
      a.peer ? reinterpret_cast<unsigned*>(a.peer + 6 * A) + (DIR ? nblk : 0) : nullptr;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase = 0;

  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int n = (int)(blk / a.nbpr);
    const int m0 = (int)(blk % a.nbpr) * BM;
    const int cols = min(BM, a.ncols - m0);
    const uint32_t rowbytes = (uint32_t)(((cols + 1) & ~1) * 8);
    const long long boff = (long long)n * a.ld + m0;
    auto chunk_of = [&](int task) { return DIR ? nchunk - 1 - task : task; };
    auto issue = [&](int c, int s) {
      const int l0 = c * K, nl = min(K, a.nzl - l0);
      mbar_arrive_expect_tx(&bar[s], 2 * nl * rowbytes + (uint32_t)(2 * nl * 12 * 8));
      for (int i = 0; i < nl; ++i) {
        const long long off = boff + (long long)(l0 + i) * a.ps;
        bulk_g2s(&sdat[s][0][i][0], a.wr + off, rowbytes, &bar[s]);
        bulk_g2s(&sdat[s][1][i][0], a.wi + off, rowbytes, &bar[s]);
      }
      bulk_g2s(&scoef[s][0][0], a.coefr + (long long)(a.z0 + l0) * 12, (uint32_t)(nl * 12 * 8),
               &bar[s]);
      bulk_g2s(&scoef[s][1][0], a.coefi + (long long)(a.z0 + l0) * 12, (uint32_t)(nl * 12 * 8),
               &bar[s]);
    };
    const bool live = tid < cols;
    const int m = m0 + tid;
    const long long idx = (long long)n * a.ld + m;
    const double cxv = __ldg(a.cx + n);
    const double cyv = live ? __ldg(a.cy + m) : 0.0;
    const double cxy = cxv * cyv;
    double* ck = a.cpk + boff + tid;
    auto lam = [&](int s, int i, int k) -> cz2 {
      return {eig_cz(&scoef[s][0][i * 12 + 4 * k], cxv, cyv, cxy),
              eig_cz(&scoef[s][1][i * 12 + 4 * k], cxv, cyv, cxy)};
    };
    if (tid == 0) {
      issue(chunk_of(0), 0);
      if (nchunk > 1) issue(chunk_of(1), 1);
    }
    cz2 c = {0.0, 0.0}, x = {0.0, 0.0};
    const bool wait_in = DIR ? has_next : has_prev;
    if (wait_in) {
      if (tid == 0) wait_block(flags_mine + blk, a.epoch, a.timeout_ns, a.xerr, DIR ? 2u : 1u);
      __syncthreads();
      if (live) {
        if (DIR) {
          x = {__ldcg(a.mine + 4 * A + idx), __ldcg(a.mine + 5 * A + idx)};
        } else {
          x = {__ldcg(a.mine + idx), __ldcg(a.mine + A + idx)};
          c = {__ldcg(a.mine + 2 * A + idx), __ldcg(a.mine + 3 * A + idx)};
        }
      }
    }
    auto cp_below = [&](int cidx) -> cz2 {
      if (!live) return {0.0, 0.0};
      if (cidx > 0)
        return {ck[(long long)(2 * (cidx - 1)) * a.ps], ck[(long long)(2 * (cidx - 1) + 1) * a.ps]};
      if (has_prev) return {__ldcg(a.mine + 2 * A + idx), __ldcg(a.mine + 3 * A + idx)};
      return {0.0, 0.0};
    };
    cz2 cbelow = DIR ? cp_below(chunk_of(0)) : cz2{0.0, 0.0};
    for (int task = 0; task < nchunk; ++task) {
      const int s = task % S;
      if (tid == 0 && task + 2 < nchunk) {
        bulk_wait_read<0>();
        fence_proxy_async_smem();
        issue(chunk_of(task + 2), (task + 2) % S);
      }
      mbar_wait(&bar[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const int cidx = chunk_of(task);
      const int l0 = cidx * K, nl = min(K, a.nzl - l0);
      if (DIR == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i < nl) {
            const int l = a.z0 + l0 + i;
            const cz2 lo = lam(s, i, 0), di = lam(s, i, 1), up = lam(s, i, 2);
            const cz2 den = (l == 0) ? di : zfms2(di, lo, c);
            double n2;
            const cz2 rr = zrcp2(den, n2);
            if (live && !(n2 >= a.thr2)) {
              const unsigned long long key =
                  ((unsigned long long)l * (unsigned long long)a.ncols + (unsigned long long)m) *
                      (unsigned long long)a.nrows +
                  (unsigned long long)n;
              atomicMin(a.err, key);
            }
            const cz2 f = {sdat[s][0][i][tid], sdat[s][1][i][tid]};
            x = zmul2((l == 0) ? f : zfms2(f, lo, x), rr);
            sdat[s][0][i][tid] = x.r;
            sdat[s][1][i][tid] = x.i;
            if (l < a.nz - 1) {
              c = zmul2(up, rr);
              if (i == K - 1 && live) {
                ck[(long long)(2 * cidx) * a.ps] = c.r;
                ck[(long long)(2 * cidx + 1) * a.ps] = c.i;
              }
            }
          }
        }
      } else {
        cz2 cprev = cbelow;
        if (task + 1 < nchunk) cbelow = cp_below(chunk_of(task + 1));
        cz2 cb[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int l = a.z0 + l0 + i;
          if (i < nl && l < a.nz - 1) {
            const cz2 di = lam(s, i, 1);
            const cz2 dl = (l == 0) ? di : zfms2(di, lam(s, i, 0), cprev);
            double n2;
            cprev = zmul2(lam(s, i, 2), zrcp2(dl, n2));
            cb[i] = cprev;
          }
        }
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
          const int l = a.z0 + l0 + i;
          if (i < nl) {
            const cz2 f = {sdat[s][0][i][tid], sdat[s][1][i][tid]};
            if (l < a.nz - 1) {
              x = zfms2(f, cb[i], x);
              sdat[s][0][i][tid] = x.r;
              sdat[s][1][i][tid] = x.i;
            } else {
              x = f;  // top of the system: W = x'
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        fence_proxy_async_smem();
        for (int i = 0; i < nl; ++i) {
          const long long off = boff + (long long)(l0 + i) * a.ps;
          bulk_s2g(a.wr + off, &sdat[s][0][i][0], rowbytes);
          bulk_s2g(a.wi + off, &sdat[s][1][i][0], rowbytes);
        }
        bulk_commit();
      }
    }
    const bool send = DIR ? has_prev : has_next;
    if (send) {
      if (live) {
        if (DIR) {
          a.peer[4 * A + idx] = x.r;
          a.peer[5 * A + idx] = x.i;
        } else {
          a.peer[idx] = x.r;
          a.peer[A + idx] = x.i;
          a.peer[2 * A + idx] = c.r;
          a.peer[3 * A + idx] = c.i;
        }
      }
      __threadfence_system();
      __syncthreads();
      if (tid == 0) st_release_sys(flags_peer + blk, a.epoch);
    }
    if (tid == 0) bulk_wait<0>();
    __syncthreads();
  }
}

long long carry_region_doubles_z(const hfb_plan* p, long long ld, long long* nblk) {
  const long long nb = (long long)p->nx * ((p->ny + BM - 1) / BM);
  if (nblk) *nblk = nb;
  return 6LL * p->nx * ld + (2 * nb + 1) / 2;
}

int launch_thomas_carry_z(hfb_plan* p, int dir, double* re, double* im, long long ld, int z0,
                          int nzl, double* cpk, double* mine, double* peer, unsigned epoch,
                          cudaStream_t st) {
  if (!p->xerr) {
    HFB_CUDA(cudaMalloc(&p->xerr, sizeof(unsigned)));
    HFB_CUDA(cudaMemset(p->xerr, 0, sizeof(unsigned)));
  }
  CarryZArgs a;
  a.wr = re;
  a.wi = im;
  a.cpk = cpk;
  a.coefr = p->coef;
  a.coefi = p->coef_i;
  a.cx = p->cx;
  a.cy = p->cy;
  a.nzl = nzl;
  a.z0 = z0;
  a.nz = p->nz;
  a.nrows = p->nx;
  a.ncols = p->ny;
  a.nbpr = (p->ny + BM - 1) / BM;
  a.ld = ld;
  a.ps = ld * p->nx;
  a.thr2 = p->thr * p->thr;
  a.err = p->err;
  a.mine = mine;
  a.peer = peer;
  a.epoch = epoch;
  const int ms = tuning(11);
  a.timeout_ns = (unsigned long long)(ms > 0 ? ms : 30000) * 1000000ULL;
  a.xerr = p->xerr;
  const size_t sm = sizeof(double) * (size_t)3 * 2 * (K * BM + K * 12);
  auto kern = dir ? thomas_carry_z_kernel<1> : thomas_carry_z_kernel<0>;
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BM, sm));
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nrows * a.nbpr;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  kern<<<(unsigned)blocks, BM, sm, st>>>(a);
  HFB_LAUNCHED();
  return HFB_OK;
}

long long carry_region_doubles(const hfb_plan* p, long long ld, long long* nblk) {
  const long long nb = (long long)p->nx * ((p->ny + BM - 1) / BM);
  if (nblk) *nblk = nb;
  return 3LL * p->nx * ld + (2 * nb + 1) / 2;
}

int launch_thomas_carry(hfb_plan* p, int dir, double* data, long long ld, int z0, int nzl,
                        double* cpk, double* mine, double* peer, unsigned epoch,
                        cudaStream_t st) {
  if (!p->xerr) {
    HFB_CUDA(cudaMalloc(&p->xerr, sizeof(unsigned)));
    HFB_CUDA(cudaMemset(p->xerr, 0, sizeof(unsigned)));
  }
  CarryArgs a;
  a.w = data;
  a.cpk = cpk;
  a.coef = p->coef;
  a.cx = p->cx;
  a.cy = p->cy;
  a.nzl = nzl;
  a.z0 = z0;
  a.nz = p->nz;
  a.nrows = p->nx;
  a.ncols = p->ny;
  a.nbpr = (p->ny + BM - 1) / BM;
  a.ld = ld;
  a.ps = ld * p->nx;
  a.thr = p->thr;
  a.err = p->err;
  a.mine = mine;
  a.peer = peer;
  a.epoch = epoch;
  const int ms = tuning(11);
  a.timeout_ns = (unsigned long long)(ms > 0 ? ms : 30000) * 1000000ULL;
  a.xerr = p->xerr;
  a.zinv = p->zinv && tuning(31);
  a.pq = p->pq;
  // tuning key 12: CTAs per SM (0 = occupancy, 3-stage ring). Capped at one or
  // two, the ring deepens to 6 stages (the HBM-bound sweep keeps its bytes in
  // flight) and the blocks come in more, shorter waves: the pipeline bubble of
  // a rank boundary is one wave per direction.
  const int cap = tuning(12);
  const int S = (cap == 1 || cap == 2) ? SMAX : 3;
  const size_t sm = sizeof(double) * (size_t)S * (K * BM + K * 12);
  auto kern = a.zinv ? (dir ? (S == 3 ? thomas_carry_kernel<1, 3, true> : thomas_carry_kernel<1, SMAX, true>)
                            : (S == 3 ? thomas_carry_kernel<0, 3, true> : thomas_carry_kernel<0, SMAX, true>))
                     : (dir ? (S == 3 ? thomas_carry_kernel<1, 3, false> : thomas_carry_kernel<1, SMAX, false>)
                            : (S == 3 ? thomas_carry_kernel<0, 3, false> : thomas_carry_kernel<0, SMAX, false>));
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BM, sm));
  if (cap > 0) per_sm = std::min(per_sm, cap);
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nrows * a.nbpr;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  kern<<<(unsigned)blocks, BM, sm, st>>>(a);
  HFB_LAUNCHED();
  return HFB_OK;
}

int launch_thomas_carry_vranks(hfb_plan* p, int dir, int nranks, double* const* data,
                               long long ld, const int* z0s, const int* nzls,
                               double* const* cpks, double* const* regions, unsigned epoch,
                               cudaStream_t st) {
  if (!p->xerr) {
    HFB_CUDA(cudaMalloc(&p->xerr, sizeof(unsigned)));
    HFB_CUDA(cudaMemset(p->xerr, 0, sizeof(unsigned)));
  }
  std::vector<CarryArgs> host(nranks);
  const int ms = tuning(11);
  for (int r = 0; r < nranks; ++r) {
    CarryArgs& a = host[r];
    memset(&a, 0, sizeof(a));
    a.w = data[r];
    a.cpk = cpks[r];
    a.coef = p->coef;
    a.cx = p->cx;
    a.cy = p->cy;
    a.nzl = nzls[r];
    a.z0 = z0s[r];
    a.nz = p->nz;
    a.nrows = p->nx;
    a.ncols = p->ny;
    a.nbpr = (p->ny + BM - 1) / BM;
    a.ld = ld;
    a.ps = ld * p->nx;
    a.thr = p->thr;
    a.err = p->err;
    a.mine = regions[r];
    a.peer = dir == 0 ? (r + 1 < nranks ? regions[r + 1] : nullptr)
                      : (r > 0 ? regions[r - 1] : nullptr);
    a.epoch = epoch;
    a.timeout_ns = (unsigned long long)(ms > 0 ? ms : 30000) * 1000000ULL;
    a.xerr = p->xerr;
    a.zinv = p->zinv && tuning(31);
    }
  constexpr int S = 3;
  const size_t sm = sizeof(double) * (size_t)S * (K * BM + K * 12);
  auto kern = host[0].zinv ? (dir ? thomas_carry_vranks_kernel<1, S, true> : thomas_carry_vranks_kernel<0, S, true>)
                           : (dir ? thomas_carry_vranks_kernel<1, S, false> : thomas_carry_vranks_kernel<0, S, false>);
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BM, sm));
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)p->nx * ((p->ny + BM - 1) / BM);
  int per = (int)std::min<long long>(work, (long long)sms * per_sm / nranks);
  if (per < 1) return HFB_ERR_ARGUMENT;  // more ranks than co-resident CTAs
  CarryArgs* dargs = nullptr;
  HFB_CUDA(cudaMalloc(&dargs, sizeof(CarryArgs) * nranks));
  HFB_CUDA(cudaMemcpy(dargs, host.data(), sizeof(CarryArgs) * nranks, cudaMemcpyHostToDevice));
  void* args[] = {&dargs, &per};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(nranks * per),
                                                    dim3(BM), args, sm, st);
  HFB_LAUNCHED();
  const cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFree(dargs);
  if (e != cudaSuccess || e2 != cudaSuccess) return HFB_ERR_CUDA;
  return HFB_OK;
}

}  // namespace hfb

// ------------------------------------------------------------------ C-ABI
using namespace hfb;

extern "C" int hfb_carry_layout(hfb_plan* p, int ld, long long* region_doubles, int* blocks) {
  if (!p || ld < p->ny || (ld & 1)) return HFB_ERR_ARGUMENT;
  long long nb = 0;
  const long long r = carry_region_doubles(p, ld, &nb);
  if (region_doubles) *region_doubles = r;
  if (blocks) *blocks = (int)nb;
  return HFB_OK;
}

extern "C" int hfb_zsolve_carry(hfb_plan* p, int dir, double* modes, int ld, int z0, int nzl,
                                void* cp_work, double* mine, double* peer, uint32_t epoch,
                                void* stream) {
  const NvtxRange nvtx_("hfb_zsolve_carry");
  if (!p || !modes || !cp_work || !mine || ld < p->ny || (ld & 1) || (dir != 0 && dir != 1))
    return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;
  if (z0 < 0 || nzl < 1 || z0 + nzl > p->nz) return HFB_ERR_RANGE;
  const bool needs_peer = dir == 0 ? z0 + nzl < p->nz : z0 > 0;
  if (needs_peer != (peer != nullptr)) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas_carry(p, dir, modes, ld, z0, nzl, (double*)cp_work, mine, peer, epoch,
                             (cudaStream_t)stream);
}

extern "C" int hfb_zsolve_carry_vranks(hfb_plan* p, int dir, int nranks, double* const* modes,
                                       int ld, const int* z0s, const int* nzls,
                                       void* const* cp_works, double* const* regions,
                                       uint32_t epoch, void* stream) {
  const NvtxRange nvtx_("hfb_zsolve_carry_vranks");
  if (!p || !modes || !z0s || !nzls || !cp_works || !regions || nranks < 1 || ld < p->ny ||
      (ld & 1) || (dir != 0 && dir != 1))
    return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;
  int next = 0;
  for (int r = 0; r < nranks; ++r) {  // consecutive slabs covering the plan's levels
    if (!modes[r] || !cp_works[r] || !regions[r] || z0s[r] != next || nzls[r] < 1)
      return HFB_ERR_RANGE;
    next += nzls[r];
  }
  if (next != p->nz) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas_carry_vranks(p, dir, nranks, modes, ld, z0s, nzls,
                                    reinterpret_cast<double* const*>(cp_works), regions, epoch,
                                    (cudaStream_t)stream);
}

extern "C" int hfb_carry_layout_z(hfb_plan* p, int ld, long long* region_doubles, int* blocks) {
  if (!p || ld < p->ny || (ld & 1)) return HFB_ERR_ARGUMENT;
  long long nb = 0;
  const long long r = carry_region_doubles_z(p, ld, &nb);
  if (region_doubles) *region_doubles = r;
  if (blocks) *blocks = (int)nb;
  return HFB_OK;
}

extern "C" int hfb_zsolve_carry_z(hfb_plan* p, int dir, double* modes_re, double* modes_im,
                                  int ld, int z0, int nzl, void* cp_work, double* mine,
                                  double* peer, uint32_t epoch, void* stream) {
  const NvtxRange nvtx_("hfb_zsolve_carry_z");
  if (!p || !modes_re || !modes_im || !cp_work || !mine || ld < p->ny || (ld & 1) ||
      (dir != 0 && dir != 1))
    return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (!p->coef_i) return HFB_ERR_ARGUMENT;  // a real table: hfb_zsolve_carry
  if (z0 < 0 || nzl < 1 || z0 + nzl > p->nz) return HFB_ERR_RANGE;
  const bool needs_peer = dir == 0 ? z0 + nzl < p->nz : z0 > 0;
  if (needs_peer != (peer != nullptr)) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas_carry_z(p, dir, modes_re, modes_im, ld, z0, nzl, (double*)cp_work, mine,
                               peer, epoch, (cudaStream_t)stream);
}

extern "C" int hfb_carry_check(hfb_plan* p, void* stream, int* code) {
  if (!p) return HFB_ERR_ARGUMENT;
  if (code) *code = 0;
  if (!p->xerr) return HFB_OK;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned v = 0;
  HFB_CUDA(cudaMemcpyAsync(&v, p->xerr, sizeof(v), cudaMemcpyDeviceToHost, st));
  HFB_CUDA(cudaStreamSynchronize(st));
  if (!v) return HFB_OK;
  HFB_CUDA(cudaMemsetAsync(p->xerr, 0, sizeof(unsigned), st));
  HFB_CUDA(cudaStreamSynchronize(st));
  if (code) *code = (int)v;
  return HFB_ERR_EXCHANGE;
}

// CUDA IPC of a carry region that lives inside a larger allocation (a torch
// caching-allocator block): the handle names the allocation, `offset` the
// region inside it.
static CUresult (*address_range())(CUdeviceptr*, size_t*, CUdeviceptr) {
  static CUresult (*fn)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r) ==
            cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(q);
  }
  return fn;
}

extern "C" int hfb_ipc_handle(const void* ptr, void* handle, long long* offset) {
  if (!ptr || !handle || !offset) return HFB_ERR_ARGUMENT;
  auto range = address_range();
  if (!range) return HFB_ERR_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return HFB_ERR_ARGUMENT;
  cudaIpcMemHandle_t h;
  HFB_CUDA(cudaIpcGetMemHandle(&h, (void*)base));
  std::memcpy(handle, &h, sizeof(h));
  *offset = (long long)((CUdeviceptr)ptr - base);
  return HFB_OK;
}

extern "C" int hfb_ipc_open(const void* handle, long long offset, void** ptr) {
  if (!handle || !ptr || offset < 0) return HFB_ERR_ARGUMENT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  HFB_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = (char*)base + offset;
  return HFB_OK;
}

extern "C" int hfb_ipc_close(void* ptr, long long offset) {
  if (!ptr) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaIpcCloseMemHandle((char*)ptr - offset));
  return HFB_OK;
}
