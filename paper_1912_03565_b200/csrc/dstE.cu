// DST-I along lines with the register-resident engine (fftE.cuh).
//
// Persistent CTAs, each holding NF transform groups (one group = M/16
// threads). A batch is one plane's block of W = 2NF consecutive lines (pair k
// = lines (2k, 2k+1), never straddling a plane). The next batch is prefetched
// into shared memory by the TMA engine while the current one is transformed
// (mbarrier, double-buffered stages), so HBM latency overlaps the arithmetic.
//
// Input modes:
//   ROW, TRAN : lines are contiguous rows, fetched with 1D bulk copies. Rows
//               need not be 16-byte aligned: the copy starts at the aligned
//               address below the row and the consumer skips the leading
//               element; a copy that would read past the end of the source is
//               shortened and thread 0 patches the last element.
//   TLOAD     : lines are COLUMNS of a padded (plane, pos, line) array, fetched
//               as 3D tensor boxes [pos][W] (cp.async.bulk.tensor); the
//               transposition happens in the TMA engine and each thread reads
//               its line pair as one double2 per position.
// Output (staged through shared memory as (line 2f, line 2f+1) double2 pairs,
// XOR-swizzled so both the per-thread segment writes and the reads are
// conflict-free):
//   ROW, TLOAD : out[plane][line][pos] — each group stores its own two lines;
//   TRAN       : out[plane][pos][line] — lines become columns; consecutive
//                threads store consecutive (pos, pair) double2 values.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fftE.cuh"
#include "tma.cuh"

namespace hfb {

// Dst16Call::mode. kYF = the y-pass of the one-call solve fused with the
// forward Thomas sweep: TLOAD input, then per mode x' = (F - lo x)/den, c =
// up/den carried across levels, x' out by tensor store, c checkpointed.
//
// kYF2 / kYB = the wavefront-fused z-solve of the one-call solve:
//   kYF2: TLOAD y-pass of (plane l, column block g), then the forward
//         elimination of its modes with the carries (x', cp at level l - 1) read
//         from the previous level's outputs in L2 (written by item (l - 1, g),
//         published by flags[g] = l); x' and cp leave by plain stores into the
//         (l, n, m) volumes S2 and CP, then flags[g] = l + 1.
//   kYB : ROW inverse y-pass over planes in DESCENDING order; before the
//         transform the staged x' rows of line pair k become W = x' - cp W(l+1)
//         with W(l+1) from the carry plane wc (item (l + 1, k), published by
//         flags[k] = n_z - 1 - l); W(l) goes back to wc, then flags[k] = n_z - l.
// Items are interleaved over persistent, co-resident CTAs in increasing order,
// and an item waits only for an item G (the items per plane) before it, so the
// wait always ends (the smallest unfinished item never waits on a later one).
// The arithmetic is thomas_tma_kernel's expression for expression: bitwise equal.
// kRowS = ROW whose input lines are split over exchange blocks (Dst16Call::split_*):
// every staged row arrives as sp_parts bulk copies of sp_kp doubles.
enum { kRow = 0, kTran = 1, kTload = 2, kYF = 3, kYF2 = 4, kYB = 5, kRowS = 6 };

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
  int nrow, ppp, G;       // lines per plane, pairs per plane, line blocks per plane
  long long in_ld, in_ps, out_ld, out_ps;
  int N, NF, logNF;       // line length, groups per CTA, log2(NF)
  int rowslot;            // doubles per staged input row (even, >= N + 4)
  int gbuf;               // doubles per group buffer (== 16/NF mod 16)
  int stage;              // doubles per stage (multiple of 128: 1-KB aligned swizzle atoms)
  int nbox, boxn;         // TLOAD: boxes per batch and their extent along the line
  int vec_out;            // TRAN: (line 2k, 2k+1) pairs are 16-byte aligned in dst
  int tstore;             // ROW/TLOAD: outputs leave by TMA tensor stores (omap)
  int pbulk;              // ROW/TLOAD into packed rows (ld = N): 1D bulk stores of row pairs
  int indep;              // ROW with tensor stores: the groups of a CTA run decoupled (own
                          // prefetch, mbarrier and tensor store; named-barrier syncs only)
  int ustore;             // ROW/TLOAD into packed rows (ld = N): a line pair is one run of 2N
                          // doubles; its full 128-byte rows leave by a 2D tensor store of the
                          // destination viewed as flat rows of 16 (umap: 2N/16-row box,
                          // omap: one row less), the <= 15-element head and tail by thread
                          // stores
  // kYF: forward Thomas sweep (thomas_tma.cu arithmetic) on the y-pass outputs
  const double* coef;     // [l][k][(4a, 2b, 2c, d)]
  const double* cx;       // per line (x-mode)
  const double* cy;       // per position (y-mode)
  double thr;
  unsigned long long* err;
  double* ck;             // cp checkpoints (l / 8, n, m) at levels 8q + 7
  long long ck_ld, ck_ps;
  int nz_total, ny_total, nx_total;
  int g0;                 // first line block of this launch
  int max_per_sm;         // cap on resident CTAs per SM (0 = occupancy)
  // kYF2 / kYB: per column block (kYF2) or line pair (kYB) level counters, the
  // back substitution's W carry plane (n, m) of row stride ck_ld, and the
  // descending plane order of kYB
  unsigned* flags;
  double* wc;
  int desc;
  int dbg;  // measurement only (tuning key 22): 1 no waits, 2 acq_rel fences, 4 no fences
  int late;               // issue the next batch's prefetch after this batch's pre-processing
                          // (tuning key 29) instead of before waiting for this batch
  int packed;             // tensor stores through a 5D map of the exchange blocks (omap)
  int sp_parts, sp_kp;    // kRowS: pieces per input line and their length
  long long sp_bstride;   // kRowS: doubles between the blocks of consecutive pieces
  int gshift;             // log2(G) when G is a power of two, else -1
  long long per;          // batches per CTA (one contiguous run), 0 = interleaved
  int run;                // > 1: interleaved runs of `run` consecutive batches
  int runshift;           // log2(run) when run is a power of two > 1, else 0
};

constexpr int kMaxRows = 16;  // 2 * NF

struct BatchMeta {
  long long plane[2];
  int row[2][kMaxRows];    // line index within the plane, -1 if absent
  int delta[2][kMaxRows];  // staged-row offset (doubles) of element 0 (ROW/TRAN)
};

// Batch `it` of this CTA: interleaved (b = blockIdx + it * grid), interleaved
// runs of a.run consecutive batches (a TLOAD CTA then reads the neighbouring
// columns of the 128-byte lines its previous box fetched while they are still
// in L2), or one contiguous run of a.per batches per CTA.
__device__ __forceinline__ bool batch_of(const StreamArgs& a, long long it, long long& plane,
                                         int& g) {
  long long b;
  if (a.per > 0) {
    if (it >= a.per) return false;
    b = (long long)blockIdx.x * a.per + it;
  } else if (a.runshift > 0) {  // runs of 2^runshift batches
    b = ((((it >> a.runshift) * gridDim.x + blockIdx.x)) << a.runshift) + (it & (a.run - 1));
  } else if (a.run > 1) {
    b = ((it / a.run) * gridDim.x + blockIdx.x) * a.run + it % a.run;
  } else {
    b = blockIdx.x + it * gridDim.x;
  }
  if (b >= (long long)a.nz * a.G) return false;
  long long q;
  int r;
  if (a.gshift >= 0) {  // G a power of two (every power-of-two line count)
    q = b >> a.gshift;
    r = (int)b & (a.G - 1);
  } else {
    q = b / a.G;
    r = (int)(b % a.G);
  }
  plane = a.desc ? a.z0 + a.nz - 1 - q : a.z0 + q;
  g = a.g0 + r;
  return true;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// spin until *p >= v (acquire); the caller then barriers its threads. The wait
// always ends by construction (see kYF2 / kYB); a broken invariant traps after
// 20 s (a launch failure) instead of spinning forever.
__device__ __forceinline__ void fence_gpu(int dbg) {
  if (dbg & 4) return;
  if (dbg & 2)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else
    __threadfence();
}
__device__ __forceinline__ void wait_level(const unsigned* p, unsigned v, int dbg) {
  if (dbg & 1) return;
  if (ld_acquire_gpu(p) < v) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_gpu(p) < v) {
      __nanosleep(64);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 20000000000ull) __trap();
    }
  }
  fence_gpu(dbg);
}
__device__ __forceinline__ double2 ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// E = 16: up to 128 threads (two line pairs of M = 1024), 3 CTAs per SM;
// E = 32: up to 64 threads (one warp per pair) and the full register budget.
// v'[j] = v[(j + r) mod Q] for a per-thread r: log2(Q) select stages (no
// dynamic register indexing), so thread t can write its segment's elements in
// a t-rotated order — distinct banks across the warp in a natural row layout.
template <int Q>
__device__ __forceinline__ void rotate_left(double (&v)[Q], int r) {
#pragma unroll
  for (int b = 1; b < Q; b <<= 1) {
    const bool on = (r & b) != 0;
    double tmp[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) tmp[j] = v[(j + b) % Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) v[j] = on ? tmp[j] : v[j];
  }
}

// M = 2048 column/transposing passes: two line pairs per CTA (W = 4 lines,
// 32-byte box rows and column chunks) at 256 threads, one CTA per SM.
template <int P, int E, int MODE>
constexpr int kMaxThreads = (E == 32 && (1 << P) <= 2048)                  ? 64
                            : (E == 16 && P == 11 && (MODE == kTran || MODE == kTload)) ? 256
                                                                                : 128;
template <int P, int E, int MODE>
constexpr int kMinBlocks = kMaxThreads<P, E, MODE> == 256 ? 1 : MODE == kYF ? 2 : 3;

template <int P, int E, int MODE>
__global__ void __launch_bounds__(kMaxThreads<P, E, MODE>, (kMinBlocks<P, E, MODE>))
    dstE_stream_kernel(StreamArgs a, FftArgs c, const __grid_constant__ CUtensorMap tmap,
                       const __grid_constant__ CUtensorMap omap,
                       const __grid_constant__ CUtensorMap umap) {
  extern __shared__ __align__(16) double sm_raw[];
  __shared__ BatchMeta meta;
  constexpr int M = FE<P, E>::M, T = FE<P, E>::T, SEG = FE<P, E>::SEG, Q = 2 * SEG;
  constexpr int LQ = FE<P, E>::LE;  // log2(Q)
  // 1-KB aligned base (swizzle atoms of the TLOAD boxes); offset arithmetic on
  // the shared array keeps every access an LDS/STS (no generic loads)
  double* sm = sm_raw + (((smem_u32(sm_raw) + 1023u) & ~1023u) - smem_u32(sm_raw)) / 8;
  const int f = threadIdx.x / T, t = threadIdx.x - f * T;
  double2* wsum = reinterpret_cast<double2*>(sm + 2LL * a.stage);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsum + (blockDim.x / 32 + 1));
  auto gbuf = [&](int s, int g) { return sm + (long long)s * a.stage + (long long)g * a.gbuf; };
  const int W = 2 * a.NF;
  constexpr bool TL = (MODE == kTload || MODE == kYF || MODE == kYF2);
  // kYF: c carried per mode, thread-major [group][line][j][t]; cy permuted
  // to [j][t] (thread t's position Q t + j)
  double* ycs = sm + 2LL * a.stage + 2 * (blockDim.x / 32 + 1) + 2;
  double* ycy = ycs + 2LL * a.NF * M;
  double yx[2][Q];  // kYF: x carried per mode
  if constexpr (MODE == kYF) {
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      const int j = i / T, tt = i - (i / T) * T, m = Q * tt + j;
      ycy[i] = m < a.ny_total ? __ldg(a.cy + m) : 0.0;
    }
#pragma unroll
    for (int L = 0; L < 2; ++L)
#pragma unroll
      for (int j = 0; j < Q; ++j) yx[L][j] = 0.0;
  }

  __shared__ uint64_t gbar[2][kMaxRows / 2];  // indep: per stage and group
  const bool indep = (MODE == kRow || MODE == kRowS || MODE == kTload || MODE == kYB) && a.indep;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    if (indep)
      for (int gg = 0; gg < a.NF; ++gg) {
        mbar_init(&gbar[0][gg], 1);
        mbar_init(&gbar[1][gg], 1);
      }
    mbar_fence_init();
  }
  __syncthreads();

  // thread 0: resolve the lines of batch `it` and start their copies into stage s
  auto issue = [&](long long it, int s) {
    long long plane;
    int g;
    batch_of(a, it, plane, g);
    meta.plane[s] = plane;
    if constexpr (TL) {
      for (int r = 0; r < W; ++r) {
        const int row = g * W + r;
        meta.row[s][r] = row < a.nrow ? row : -1;
      }
      mbar_arrive_expect_tx(&bar[s], (uint32_t)(a.nbox * a.boxn * W * 8));
      for (int b = 0; b < a.nbox; ++b)
        tensor_g2s_3d(gbuf(s, 0) + (long long)b * a.boxn * W, &tmap, g * W, b * a.boxn,
                      (int)plane, &bar[s]);
    } else if constexpr (MODE == kRowS) {
      // every present row arrives as sp_parts pieces of sp_kp doubles (16-byte
      // aligned at both ends), staged contiguously at gbuf(s, r/2) + (r&1)*rowslot + 2
      uint32_t total = 0;
      for (int r = 0; r < W; ++r) {
        const int k = g * a.NF + (r >> 1);
        const int row = 2 * k + (r & 1);
        const bool ok = k < a.ppp && row < a.nrow;
        meta.row[s][r] = ok ? row : -1;
        meta.delta[s][r] = 2;
        if (ok) total += (uint32_t)(a.sp_parts * a.sp_kp * 8);
      }
      mbar_arrive_expect_tx(&bar[s], total);
      for (int r = 0; r < W; ++r) {
        const int row = meta.row[s][r];
        if (row < 0) continue;
        const double* A = a.src + (plane * a.nrow + row) * a.sp_kp;
        double* dstrow = gbuf(s, r >> 1) + (r & 1) * a.rowslot + 2;
        for (int q = 0; q < a.sp_parts; ++q)
          bulk_g2s(dstrow + q * a.sp_kp, A + q * a.sp_bstride, (uint32_t)(a.sp_kp * 8), &bar[s]);
      }
    } else {
      // staged row r at gbuf(s, r/2) + (r&1)*rowslot + 2 (16-B aligned)
      uint32_t total = 0;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) mbar_arrive_expect_tx(&bar[s], total);
#pragma unroll 1
        for (int r = 0; r < W; ++r) {
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
    }
  };

  // indep (ROW): the leader of group f brings the group's two rows of batch `it`
  // into its own buffer of stage s, completing on gbar[s][f]
  auto issue_rows = [&](long long it, int s) {
    long long plane;
    int g;
    batch_of(a, it, plane, g);
    if constexpr (MODE == kRowS) {
      uint32_t tot = 0;
      for (int r = 2 * f; r < 2 * f + 2; ++r) {
        const int k = g * a.NF + (r >> 1);
        const int row = 2 * k + (r & 1);
        const bool ok = k < a.ppp && row < a.nrow;
        meta.row[s][r] = ok ? row : -1;
        meta.delta[s][r] = 2;
        if (ok) tot += (uint32_t)(a.sp_parts * a.sp_kp * 8);
      }
      mbar_arrive_expect_tx(&gbar[s][f], tot);
      for (int r = 2 * f; r < 2 * f + 2; ++r) {
        const int row = meta.row[s][r];
        if (row < 0) continue;
        const double* A = a.src + (plane * a.nrow + row) * a.sp_kp;
        double* dstrow = gbuf(s, f) + (r & 1) * a.rowslot + 2;
        for (int q = 0; q < a.sp_parts; ++q)
          bulk_g2s(dstrow + q * a.sp_kp, A + q * a.sp_bstride, (uint32_t)(a.sp_kp * 8),
                   &gbar[s][f]);
      }
      return;
    }
    uint32_t total = 0;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) mbar_arrive_expect_tx(&gbar[s][f], total);
#pragma unroll 1
      for (int r = 2 * f; r < 2 * f + 2; ++r) {
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
        double* dstrow = gbuf(s, f) + (r & 1) * a.rowslot + 2;
        if (pass == 0) {
          total += S;
          meta.row[s][r] = row;
          meta.delta[s][r] = 2 + d;
          if (cut) dstrow[d + a.N - 1] = __ldg(A + a.N - 1);  // not covered by the copy
        } else {
          bulk_g2s(dstrow, A16, S, &gbar[s][f]);
        }
      }
    }
  };

  // indep (TLOAD): the leader of group f brings the group's two columns of batch
  // `it` as unswizzled [pos][2 lines] boxes into its own buffer of stage s
  auto issue_box = [&](long long it, int s) {
    long long plane;
    int g;
    batch_of(a, it, plane, g);
    for (int r = 2 * f; r < 2 * f + 2; ++r) {
      const int row = g * W + r;
      meta.row[s][r] = row < a.nrow ? row : -1;
    }
    mbar_arrive_expect_tx(&gbar[s][f], (uint32_t)(a.nbox * a.boxn * 2 * 8));
    for (int b = 0; b < a.nbox; ++b)
      tensor_g2s_3d(gbuf(s, f) + (long long)b * a.boxn * 2, &tmap, g * W + 2 * f, b * a.boxn,
                    (int)plane, &gbar[s][f]);
  };

  EngineTw<P, E> etw;
  engine_tw<P, E>(c.tw, c.sn, t, etw);
  int s = 0;
  uint32_t phase0 = 0, phase1 = 0;
  {
    long long pl;
    int g;
    if (indep) {
      if (t == 0 && batch_of(a, 0, pl, g)) {
        if constexpr (TL) issue_box(0, 0); else issue_rows(0, 0);
      }
    } else if (threadIdx.x == 0 && batch_of(a, 0, pl, g)) {
      issue(0, 0);
    }
  }
  // Prefetch batch it + 1 into the other stage. Its buffer's previous batch
  // (it - 1) must have been read out by its store: issued right at the start
  // of batch it, the leader waits for the store committed a moment before
  // while the rest of its group (or CTA) goes on, then waits for the leader;
  // issued after the pre-processing (a.late) the store has long finished and
  // the copy still has the FFT, post-processing and store of batch it to land.
  auto prefetch_next = [&](long long it) {
    {
      long long pl2;
      int g2;
      if (indep) {
        if (t == 0 && batch_of(a, it + 1, pl2, g2)) {
          bulk_wait_read<0>();  // this group's batch it-1 store read its buffer of stage s^1
          fence_proxy_async_smem();
          if constexpr (TL) issue_box(it + 1, s ^ 1); else issue_rows(it + 1, s ^ 1);
        }
      } else if (threadIdx.x == 0 && batch_of(a, it + 1, pl2, g2)) {
        if (a.tstore || a.pbulk || a.ustore) bulk_wait_read<0>();  // batch it-1's stores read stage s^1
        fence_proxy_async_smem();
        issue(it + 1, s ^ 1);
      }
    }
  };
  for (long long it = 0;; ++it) {
    long long plane;
    int g;
    if (!batch_of(a, it, plane, g)) break;
    if (!a.late) prefetch_next(it);
    mbar_wait(indep ? &gbar[s][f] : &bar[s], s == 0 ? phase0 : phase1);
    if (s == 0) phase0 ^= 1; else phase1 ^= 1;

    double* gb = gbuf(s, f);
    const int row0 = meta.row[s][2 * f], row1 = meta.row[s][2 * f + 1];
    const bool v0 = row0 >= 0, v1 = row1 >= 0;

    double2 v[E];
    if constexpr (TL) {
      // box [pos][W]: a_e of lines (2f, 2f+1) is the double2 at pos e - 1
      // (absent lines and positions >= N were zero-filled by the TMA engine)
      // (the box is swizzled: 16-byte granule g sits at g ^ ((g >> 3) & (NF - 1)))
      if (indep) {  // the group's own [pos][2 lines] box, unswizzled
        const double2* bx = reinterpret_cast<const double2*>(gb);
        dstE_pre<P, E>(v, c.sn, etw, t,
                       [&](int e) -> double2 { return bx[(e + M - 1) & (M - 1)]; });
        group_sync<T>(f);
        if (a.late) prefetch_next(it);
      } else {
        const double2* bx = reinterpret_cast<const double2*>(gbuf(s, 0));
        if (E == 16 && T >= 8 && a.NF == 2) {
          // granule 2 pos + f of position pos = e - 1, XOR term bit 2 of pos: for
          // e = t + T i that bit is bit 2 of t - 1, for e = M - t - T i bit 2 of
          // M - 1 - t (T i leaves bit 2 alone): two per-thread bases plus
          // compile-time offsets +-2 T i (the same slots as the generic form
          // below; e = 0 and e = M keep it — their values are selected away)
          const int lo = t - 1, hi = M - 1 - t;
          const double2* pl = bx + 2 * lo + (f ^ ((lo >> 2) & 1));
          const double2* ph = bx + 2 * hi + (f ^ ((hi >> 2) & 1));
          dstE_pre_idx<P, E>(v, c.sn, etw, t, [&](int i, bool mirror) -> double2 {
            if (i == 0) {  // e = t (t = 0: unused) or e = M - t (t = 0: unused)
              const int e = mirror ? M - t : t;
              const int gr = ((e + M - 1) & (M - 1)) * 2 + f;
              return bx[gr ^ ((gr >> 3) & 1)];
            }
            return mirror ? ph[-2 * T * i] : pl[2 * T * i];
          });
        } else {
          dstE_pre<P, E>(v, c.sn, etw, t, [&](int e) -> double2 {
            const int gr = ((e + M - 1) & (M - 1)) * a.NF + f;
            return bx[gr ^ ((gr >> 3) & (a.NF - 1))];
          });
        }
        __syncthreads();  // the box interleaves all groups' lines
        if (a.late) prefetch_next(it);
      }
    } else {
      if constexpr (MODE == kYB) {
        // back substitution on the staged x' rows of this group's line pair:
        // W(l) = x'(l) - cp(l) W(l+1) (thomas_tma_kernel's fma), W(l) -> wc
        const int l = (int)plane, nzt = a.nz_total;
        const int pair = g * a.NF + f;
        if (l < nzt - 1) {
          if (t == 0) wait_level(a.flags + pair, (unsigned)(nzt - 1 - l), a.dbg);
          group_sync<T>(f);
        }
        // W(l) = x'(l) - cp(l) W(l + 1) on coalesced 16-byte lanes of each line
#pragma unroll
        for (int L = 0; L < 2; ++L) {
          const int n = L ? row1 : row0;
          if (n < 0) continue;
          double* row = gb + L * a.rowslot + meta.delta[s][2 * f + L];  // position m at row[m]
          double* wr = a.wc + (long long)n * a.ck_ld;
          const double* cr = a.ck + (long long)l * a.ck_ps + (long long)n * a.ck_ld;
#pragma unroll 4
          for (int u = t; 2 * u < a.N; u += T) {
            const int m = 2 * u;
            double2 x = *reinterpret_cast<const double2*>(row + m);
            if (l < nzt - 1) {
              const double2 c2 = __ldg(reinterpret_cast<const double2*>(cr + m));
              const double2 w2 = ldcg2(wr + m);
              x.x = fma(-c2.x, w2.x, x.x);
              x.y = fma(-c2.y, w2.y, x.y);
            }
            *reinterpret_cast<double2*>(wr + m) = x;
            *reinterpret_cast<double2*>(row + m) = x;
          }
        }
        group_sync<T>(f);
        if (t == 0) {
          fence_gpu(a.dbg);
          st_release_gpu(a.flags + pair, (unsigned)(nzt - l));
        }
      }
      const double* r0 = gb + meta.delta[s][2 * f] - 1;  // a_e at r0[e]
      const double* r1 = gb + a.rowslot + meta.delta[s][2 * f + 1] - 1;
      if constexpr (T >= 32) {
        // (groups of whole warps: the group barrier below is legal in a branch
        // that is uniform per group)
        if (!(v0 && v1)) {
          // an absent line (the odd line out at the end of a plane) is a staged
          // row of zeros, so the loads below carry no per-element select
          if (!v0)
            for (int e = 1 + t; e <= a.N; e += T) const_cast<double*>(r0)[e] = 0.0;
          if (!v1)
            for (int e = 1 + t; e <= a.N; e += T) const_cast<double*>(r1)[e] = 0.0;
          group_sync<T>(f);
        }
        dstE_pre<P, E>(v, c.sn, etw, t,
                       [&](int e) -> double2 { return make_double2(r0[e], r1[e]); });
      } else {
        dstE_pre<P, E>(v, c.sn, etw, t, [&](int e) -> double2 {
          return make_double2(v0 ? r0[e] : 0.0, v1 ? r1[e] : 0.0);
        });
      }
      group_sync<T>(f);  // staged rows consumed: the group buffer becomes FFT scratch
      if (a.late) prefetch_next(it);
    }
    double2* sb = reinterpret_cast<double2*>(gb);
    fftE_forward<P, E>(v, sb, etw, t, f);
    double2 out[Q];
    if constexpr (MODE == kYF2) {
      dstE_post_aligned<P, E>(v, sb, wsum, c.scale, t, f, out);
      // The outputs wait in the group's scratch in the 128B-swizzled box layout
      // of the tensor-store path (conflict-free both ways), and the elimination
      // re-maps threads to modes m = t + T i: every carry load and every x' / cp
      // store is then a coalesced 256-byte warp access, and the transform's
      // registers are free for the carries.
      constexpr int NSEG = M / 16;
      auto phys = [](int L, int pos) {
        const int row = L * NSEG + (pos >> 4);
        return row * 16 + 2 * (((pos >> 1) & 7) ^ (row & 7)) + (pos & 1);
      };
#pragma unroll
      for (int L = 0; L < 2; ++L)
#pragma unroll
        for (int h = 0; h < Q / 2; ++h) {
          const int pos = Q * t + 2 * h;
          *reinterpret_cast<double2*>(gb + phys(L, pos)) =
              L == 0 ? make_double2(out[2 * h].x, out[2 * h + 1].x)
                     : make_double2(out[2 * h].y, out[2 * h + 1].y);
        }
      group_sync<T>(f);
      // forward elimination at level l of the group's 2 x M modes; the carries
      // are level l - 1's outputs of the same column block
      const int l = (int)plane, nzt = a.nz_total;
      if (l > 0) {
        if (threadIdx.x == 0) wait_level(a.flags + g, (unsigned)l, a.dbg);
        __syncthreads();
      }
      const double* cwp = a.coef + (long long)l * 12;
#pragma unroll 1
      for (int L = 0; L < 2; ++L) {
        const int n = L ? row1 : row0;
        if (n < 0) continue;
        const double cxv = __ldg(a.cx + n);
        const long long o = (long long)n * a.out_ld + t;
        double* xo = a.dst + (long long)l * a.out_ps + o;
        double* co = a.ck + (long long)l * a.ck_ps + o;
        double cw[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) cw[q] = __ldg(cwp + q);
        constexpr int H = Q / 2;  // modes per carry batch
#pragma unroll 1
        for (int h = 0; h < Q; h += H) {
          double xin[H], cin[H];
          if (l > 0) {
            const double* xp = xo - a.out_ps + T * h;
            const double* cq = co - a.ck_ps + T * h;
#pragma unroll
            for (int i = 0; i < H; ++i) {
              xin[i] = __ldcg(xp + T * i);
              cin[i] = __ldcg(cq + T * i);
            }
          }
#pragma unroll
          for (int i = 0; i < H; ++i) {
            const int m = t + T * (h + i);
            const double cyv = m < a.ny_total ? __ldg(a.cy + m) : 0.0;
            const double cxy = cxv * cyv;
            (void)cxy;
            const double lo = eig_pq(cw, cxv, cyv);
            const double di = eig_pq(cw + 4, cxv, cyv);
            const double up = eig_pq(cw + 8, cxv, cyv);
            const double den = (l == 0) ? di : fma(-lo, cin[i], di);
            if (m < a.ny_total && fabs(den) < a.thr) {
              const unsigned long long key =
                  ((unsigned long long)l * (unsigned long long)a.ny_total + (unsigned long long)m) *
                      (unsigned long long)a.nx_total +
                  (unsigned long long)n;
              atomicMin(a.err, key);
            }
            const double rr = rcp_fast(den);
            const double F = gb[phys(L, m)];
            xo[T * (h + i)] = ((l == 0) ? F : fma(-lo, xin[i], F)) * rr;
            if (l < nzt - 1) co[T * (h + i)] = up * rr;
          }
        }
      }
      __syncthreads();  // every thread's x' and cp of level l are stored
      if (threadIdx.x == 0) {
        fence_gpu(a.dbg);
        st_release_gpu(a.flags + g, (unsigned)(l + 1));
      }
    } else if (MODE != kTran && (a.tstore || a.pbulk || a.ustore)) {
      // Segment-aligned outputs staged as the group's tensor box [2 lines]
      // [M/16 segments][16] in the 128B-swizzle layout (granule h of smem row r
      // at h ^ (r & 7): conflict-free, since thread t owns whole segments),
      // then one TMA tensor store per group (issued by thread 0).
      dstE_post_aligned<P, E>(v, sb, wsum, c.scale, t, f, out);
      if constexpr (MODE == kYF) {
        // forward elimination at level l for this thread's 2 x Q modes,
        // bitwise the arithmetic of thomas_tma_kernel
        const int l = (int)plane;
        double cw[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) cw[q] = __ldg(a.coef + (long long)l * 12 + q);
#pragma unroll
        for (int L = 0; L < 2; ++L) {
          const int n = L ? row1 : row0;
          const double cxv = n >= 0 ? __ldg(a.cx + n) : 0.0;
          double* cs = ycs + ((long long)(f * 2 + L) * Q) * T + t;
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            const int m = Q * t + j;
            const double cyv = ycy[j * T + t];
            const double cxy = cxv * cyv;
            (void)cxy;
            const double lo = eig_pq(cw, cxv, cyv);
            const double di = eig_pq(cw + 4, cxv, cyv);
            const double up = eig_pq(cw + 8, cxv, cyv);
            const double den = (l == 0) ? di : fma(-lo, cs[j * T], di);
            const bool live = n >= 0 && m < a.ny_total;
            if (live && fabs(den) < a.thr) {
              const unsigned long long key =
                  ((unsigned long long)l * (unsigned long long)a.ny_total + (unsigned long long)m) *
                      (unsigned long long)a.nx_total +
                  (unsigned long long)n;
              atomicMin(a.err, key);
            }
            const double rr = rcp_fast(den);
            const double F = L ? out[j].y : out[j].x;
            const double x = ((l == 0) ? F : fma(-lo, yx[L][j], F)) * rr;
            yx[L][j] = x;
            if (L) out[j].y = x; else out[j].x = x;
            if (l < a.nz_total - 1) {
              const double cc = up * rr;
              cs[j * T] = cc;
              if ((l & 7) == 7 && live)
                a.ck[(long long)(l >> 3) * a.ck_ps + (long long)n * a.ck_ld + m] = cc;
            }
          }
        }
      }
      if (a.tstore) {
        constexpr int NSEG = M / 16;
#pragma unroll
        for (int L = 0; L < 2; ++L) {
          // Q = 16: thread t owns box row L NSEG + t; granule h of it sits at
          // h ^ (row & 7): double2 slot (8 row ^ (row & 7)) ^ h
          const int rowq = L * NSEG + t;
          const int bq = (8 * rowq) ^ (rowq & 7);
#pragma unroll
          for (int h = 0; h < Q / 2; ++h) {
            const double2 val = L == 0 ? make_double2(out[2 * h].x, out[2 * h + 1].x)
                                       : make_double2(out[2 * h].y, out[2 * h + 1].y);
            if constexpr (Q == 16 && kXorAddr<P, E>) {
              sh_st2((sh_addr(gb) + 16u * (uint32_t)bq) ^ (16u * h), val);
            } else if constexpr (Q == 16) {
              reinterpret_cast<double2*>(gb)[bq ^ h] = val;
            } else {
              const int pos = Q * t + 2 * h;
              const int row = L * NSEG + (pos >> 4);
              const int phys = row * 16 + 2 * (((pos >> 1) & 7) ^ (row & 7));
              *reinterpret_cast<double2*>(gb + phys) = val;
            }
          }
        }
        fence_proxy_async_smem();
        if (indep) {
          group_sync<T>(f);
          if (t == 0) {
            if (row0 >= 0) {
              if (a.packed) tensor_s2g_5d(&omap, 0, 0, 0, row0, (int)plane, gb);
              else tensor_s2g_4d(&omap, 0, 0, row0, (int)plane, gb);
            }
            bulk_commit();
          }
        } else {
          __syncthreads();
          if (threadIdx.x == 0) {
            for (int gg = 0; gg < a.NF; ++gg) {
              const int r0 = meta.row[s][2 * gg];
              if (r0 >= 0) {
                if (a.packed) tensor_s2g_5d(&omap, 0, 0, 0, r0, (int)plane, gbuf(s, gg));
                else tensor_s2g_4d(&omap, 0, 0, r0, (int)plane, gbuf(s, gg));
              }
            }
            bulk_commit();
          }
        }
      } else if (a.ustore) {
        if constexpr (Q == 16) {
          // The group's two lines are one run of 2N doubles at flat offset o of the
          // destination; run element e sits at u = e - ha in the box of the flat
          // 128-byte rows that start at o + ha (the first 16-aligned offset). Every
          // element is staged at box row u >> 4 (128B-swizzled), head elements
          // (u < 0) in the spare row -1 and tail elements past the full rows: the
          // staging code is branch-free, and a thread's granule-aligned pairs are
          // 16-byte stores on 8 distinct bank groups per 8 lanes. The full rows leave
          // by one 2D tensor store (thread 0); the <= 15 head and tail elements by
          // plain stores from shared memory.
          const long long o = plane * a.out_ps + (long long)row0 * a.out_ld;
          const int ha = (int)((16 - (o & 15)) & 15);
          double* ub = gb + 128;  // box row 0: 1-KB aligned, row -1 below it
#pragma unroll
          for (int L = 0; L < 2; ++L) {
            const int u0 = L * a.N + Q * t - ha;
            // element u at box row u >> 4, 16-byte granule ((u >> 1) & 7) ^ (row & 7):
            // with hp = u >> 1 that is slot 2 (hp ^ ((hp >> 3) & 7)) + (u & 1) (row -1
            // included: the arithmetic shifts keep hp in [-8, -1] there)
            auto at = [&](int u) { const int hp = u >> 1;
                                   return ub + 2 * (hp ^ ((hp >> 3) & 7)) + (u & 1); };
            auto val = [&](int jj) { return L ? out[jj].y : out[jj].x; };
            const bool last = Q * t + Q > a.N;  // the segment holding the padding position
            if (!(u0 & 1)) {
#pragma unroll
              for (int jj = 0; jj < Q; jj += 2) {
                double* d = at(u0 + jj);
                if (jj < Q - 2 || !last)
                  *reinterpret_cast<double2*>(d) = make_double2(val(jj), val(jj + 1));
                else
                  *d = val(jj);
              }
            } else {
              *at(u0) = val(0);
#pragma unroll
              for (int jj = 1; jj < Q - 1; jj += 2)
                *reinterpret_cast<double2*>(at(u0 + jj)) = make_double2(val(jj), val(jj + 1));
              if (!last) *at(u0 + Q - 1) = val(Q - 1);
            }
          }
          fence_proxy_async_smem();
          const int len = (v1 ? 2 : 1) * a.N;
          const int nrows = (len - ha) >> 4;
          const int hi = (2 * a.N) >> 4;  // full rows of a pair run: hi or hi - 1
          const bool tma = v1 && (nrows == hi || nrows == hi - 1);
          if (indep) {
            group_sync<T>(f);
            if (t == 0) {
              if (tma) tensor_s2g_2d(nrows == hi ? &umap : &omap, 0, (int)((o + ha) >> 4), ub);
              bulk_commit();
            }
          } else {
            __syncthreads();
          }
          if (!indep && threadIdx.x == 0) {
            for (int gg = 0; gg < a.NF; ++gg) {
              const int r0 = meta.row[s][2 * gg];
              if (r0 < 0 || meta.row[s][2 * gg + 1] < 0) continue;
              const long long og = plane * a.out_ps + (long long)r0 * a.out_ld;
              const int hg = (int)((16 - (og & 15)) & 15);
              const int ng = (2 * a.N - hg) >> 4;
              const int frow = (int)((og + hg) >> 4);
              if (ng == hi) tensor_s2g_2d(&umap, 0, frow, gbuf(s, gg) + 128);
              else if (ng == hi - 1) tensor_s2g_2d(&omap, 0, frow, gbuf(s, gg) + 128);
            }
            bulk_commit();
          }
          if (v0) {
            double* G = a.dst + o;
            auto ld_u = [&](int u) {
              const int q = u >> 4, cc = u & 15;
              return ub[q * 16 + 2 * ((cc >> 1) ^ (q & 7)) + (cc & 1)];
            };
            if (tma) {
              if (t < ha) G[t] = ld_u(t - ha);
              const int e = ha + 16 * nrows + t;
              if (e < len) G[e] = ld_u(e - ha);
            } else {
              for (int e = t; e < len; e += T) G[e] = ld_u(e - ha);
            }
          }
        }
      } else if constexpr (Q == 16) {
        // Packed rows (ld = N): the group's two lines are one contiguous run of
        // 2N doubles. Stage it in natural order, element e at gb[d + e] with d
        // the run's 16-byte misalignment, writing in a t-rotated order; then
        // the 16-byte aligned body leaves by one 1D bulk store and the at most
        // two edge elements by plain stores.
        double* G = a.dst + plane * a.out_ps + (long long)row0 * a.out_ld;
        const int d = (int)((reinterpret_cast<uintptr_t>(G) >> 3) & 1);
        double w0[Q], w1[Q];
#pragma unroll
        for (int c = 0; c < Q; ++c) {
          w0[c] = out[c].x;
          w1[c] = out[c].y;
        }
        rotate_left<Q>(w0, t & (Q - 1));
        rotate_left<Q>(w1, t & (Q - 1));
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          const int p = Q * t + ((j + t) & (Q - 1));
          if (p < a.N) {
            gb[d + p] = w0[j];
            if (v1) gb[d + a.N + p] = w1[j];
          }
        }
        group_sync<T>(f);
        const int etot = (v1 ? 2 : 1) * a.N;
        const int nb = (etot - d) & ~1;
        if (t == 0 && v0) {
          if (d) G[0] = gb[d];
          if (d + nb < etot) G[etot - 1] = gb[d + etot - 1];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          for (int gg = 0; gg < a.NF; ++gg) {
            const int r0 = meta.row[s][2 * gg];
            if (r0 < 0) continue;
            double* Gg = a.dst + plane * a.out_ps + (long long)r0 * a.out_ld;
            const int dg = (int)((reinterpret_cast<uintptr_t>(Gg) >> 3) & 1);
            const int eg = (meta.row[s][2 * gg + 1] >= 0 ? 2 : 1) * a.N;
            const int nbg = (eg - dg) & ~1;
            if (nbg > 0) bulk_s2g(Gg + dg, gbuf(s, gg) + 2 * dg, (uint32_t)nbg * 8);
          }
          bulk_commit();
        }
      }
    } else {
      dstE_post<P, E>(v, sb, wsum, c.scale, t, f, out);
      // stage: output position p of the pair at slot swz<LQ>(p)
      double2* st2 = reinterpret_cast<double2*>(gb);
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        const int p = Q * t + j - 1;
        if (p >= 0) st2[swz<LQ>(p)] = out[j];
      }
      if constexpr (MODE == kTran) {
        __syncthreads();
        const int total = a.N << a.logNF;
        double* ob = a.dst + plane * a.out_ps;
        for (int e = threadIdx.x; e < total; e += blockDim.x) {
          const int pos = e >> a.logNF, gg = e & (a.NF - 1);
          const int r0 = meta.row[s][2 * gg];
          if (r0 < 0) continue;
          const bool has1 = meta.row[s][2 * gg + 1] >= 0;
          const double2 val =
              lds128(reinterpret_cast<const double2*>(gbuf(s, gg)) + swz<LQ>(pos));
          double* o = ob + (long long)pos * a.out_ld + r0;
          if (a.vec_out && has1) {
            *reinterpret_cast<double2*>(o) = val;
          } else {
            o[0] = val.x;
            if (has1) o[1] = val.y;
          }
        }
      } else {
        group_sync<T>(f);
        double* o0 = a.dst + plane * a.out_ps + (long long)row0 * a.out_ld;
        double* o1 = a.dst + plane * a.out_ps + (long long)row1 * a.out_ld;
        for (int p = t; p < a.N; p += T) {
          const double2 val = lds128(&st2[swz<LQ>(p)]);
          if (v0) o0[p] = val.x;
          if (v1) o1[p] = val.y;
        }
      }
    }
    if (indep)
      group_sync<T>(f);  // the group's buffer of stage s is free for its next prefetch
    else
      __syncthreads();  // stage s is free for the prefetch issued next iteration
    s ^= 1;
  }
  if ((a.tstore || a.pbulk || a.ustore) && (indep ? t == 0 : threadIdx.x == 0))
    bulk_wait<0>();  // smem valid until stored
}

bool dst16_ok(int M) { return M >= 16 && M <= 4096 && (M & (M - 1)) == 0; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// tuning knobs (hfb_set_tuning): engine width E for M >= 32 and groups per CTA
static int g_tune_E = 16;
static int g_tune_NF = 0;
static int g_tune_l2 = 2;     // TLOAD tensor-map L2 promotion: 0 none, 1 64B, 2 128B, 3 256B
static int g_tune_order = 0;  // batch order: 0 auto, 1 one run per CTA, R >= 2 runs of R
static int g_tune_tstore = 1;  // row outputs by TMA tensor stores where the layout allows
static int g_tune_overlap = 0;  // overlapped z-solve / y-pass schedule (key 6)
static int g_tune_cap_dst = 2;  // its CTA caps per SM: y-passes (key 7), z-solve (key 8)
static int g_tune_cap_th = 1;
static int g_tune_pbulk = 0;    // packed-row outputs by row-pair bulk stores (key 9; off: slower)
static int g_tune_fuse = 0;    // one-call solve: forward Thomas fused into the y-pass (off: occupancy-starved, 12 ms vs 4 + 3)
static int g_tune_cap_all = 0;  // cap on resident CTAs per SM for every DST pass (key 10; 0 = occupancy)
static int g_tune_carry_ms = 0;  // distributed z-solve: carry wait timeout in ms (key 11; 0 = 30 s)
static int g_tune_carry_cap = 0;  // distributed z-solve: CTAs per SM (key 12; 0 = occupancy)
static int g_tune_ustore = 1;  // packed-row outputs by flat-row tensor stores (key 13)
static int g_tune_indep = 1;   // ROW passes with tensor stores: decoupled groups (key 14)
static int g_tune_dmma = 1;    // dense DST-I products on the FP64 tensor cores (key 16)
static int g_tune_dense_max = 0;  // force the dense path for lines up to this length (key 17)
static int g_tune_dmma2d = 32;  // whole-plane DMMA 2D DST-I for lines up to this length (key 18)
static int g_tune_rhs_march = 32;  // 4th-order RHS operator: levels per marching CTA (key 20; 0 = gathers)
static int g_tune_thomas_smem = 1;  // one-call z-solve with whole columns in shared memory, n_z <= 256 (key 19)
// one-call solve: wavefront-fused z-solve in the y-passes (key 21). Off: measured
// 34.7 vs 22.1 ms at 1023^3 — the carry / cp loads stall the
// 12 warps per SM the register-resident engine leaves (long scoreboard 3-8 per issue)
static int g_tune_wave = 0;
static int g_tune_xsparse = 1;  // one-call z-solve stores x' once per chunk, recomputes the rest (key 23)
static int g_tune_s27 = 32;  // streamed 27-point apply / residual: levels per CTA (key 24; 0 = key 20's kernels)
static int g_tune_s27_rj = 4;  // rows per warp of the streamed 27-point kernels (key 25: 2 or 4)
static int g_tune_thomas_stages = 3;  // ring stages of the TMA z-solve (key 26: 3 or 4)
static int g_tune_s27_tile = 1;  // streamed 27-point kernels: planes staged in shared memory (key 27)
static int g_tune_late = 2;  // DST passes: prefetch after the pre-processing (key 29; 2 = flat-row-store passes)
static int g_tune_thomas_narrow = 0;  // TMA z-solve with 128-mode blocks (key 28)
static int g_tune_thomas_kc = 0;  // TMA z-solve chunks (key 30: 0 = 8 levels, 1 = 16 levels 3 stages, 2 = 16 levels 2 stages)
static int g_tune_zinv = 1;  // TMA z-solve: eigenvalues once per mode for z-invariant weights (key 31)
static int g_tune_ckcache = 1;  // one-call z-solve: cp checkpoints cached in the plan across solves (key 32)
static int g_tune_wave_dbg = 0;  // its measurement variants (key 22; wrong results for bit 1)

template <int P, int E, int MODE>
static int launch_stream(const StreamArgs& a, const FftArgs& c, const CUtensorMap& tmap,
                         const CUtensorMap& omap, const CUtensorMap& umap, int threads, size_t sm,
                         cudaStream_t st) {
  auto kern = dstE_stream_kernel<P, E, MODE>;
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                cudaSharedmemCarveoutMaxShared));
  int per_sm = 1;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, sm));
  if (a.max_per_sm > 0) per_sm = std::min(per_sm, a.max_per_sm);
  if (g_tune_cap_all > 0) per_sm = std::min(per_sm, g_tune_cap_all);
  if (getenv("HFB_DEBUG"))
    fprintf(stderr, "dstE<P=%d,E=%d,mode=%d>: %d threads, %zu B smem, %d CTAs/SM\n", P, E, MODE,
            threads, sm, per_sm);
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nz * a.G;
  long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  StreamArgs b = a;
  b.per = 0;
  b.run = 1;
  b.gshift = -1;
  if (a.G > 0 && (a.G & (a.G - 1)) == 0)
    for (b.gshift = 0; (1 << b.gshift) < a.G;) ++b.gshift;
  if (MODE == kYF) {
    // one CTA per column block, walking the levels in order (the Thomas carry)
    blocks = a.G;
  } else if (MODE == kYF2 || MODE == kYB) {
    // wavefront-fused z-solve: interleaved items over co-resident CTAs (the
    // flag waits need every CTA resident), column blocks in runs of two
    b.run = MODE == kYF2 ? 2 : 1;
  } else if (g_tune_order == 1) {
    b.per = (work + blocks - 1) / blocks;
    blocks = (work + b.per - 1) / b.per;
  } else if (g_tune_order >= 2) {
    b.run = g_tune_order;
  } else if (MODE == kTload) {
    b.run = 2;  // pairs of neighbouring column blocks (measured best at W = 4)
  }
  b.runshift = 0;
  if (b.run > 1 && (b.run & (b.run - 1)) == 0)
    while ((1 << b.runshift) < b.run) ++b.runshift;
  kern<<<(unsigned)blocks, threads, sm, st>>>(b, c, tmap, omap, umap);
  return HFB_OK;
}

template <int P, int E>
static int launch_pe(const Dst16Call& k, StreamArgs a, const FftArgs& c, cudaStream_t st) {
  using G = FE<P, E>;
  constexpr int T = G::T, M = G::M;
  const int maxt = k.mode == kTran    ? kMaxThreads<P, E, kTran>
                   : k.mode == kTload ? kMaxThreads<P, E, kTload>
                   : k.mode == kYF    ? kMaxThreads<P, E, kYF>
                   : k.mode == kYF2   ? kMaxThreads<P, E, kYF2>
                   : k.mode == kYB    ? kMaxThreads<P, E, kYB>
                                      : kMaxThreads<P, E, kRow>;
  if ((k.mode == kYF2 || k.mode == kYB) && (P > 10 || E != 16 || !k.flags || !k.cp ||
                                            !k.coef || (k.mode == kYB && !k.wc)))
    return HFB_ERR_ARGUMENT;
  int nf = std::max(1, std::min(maxt / T, kMaxRows / 2));
  if (g_tune_NF > 0) nf = std::max(1, std::min(g_tune_NF, nf));
  a.NF = 1;
  a.logNF = 0;
  while (2 * a.NF <= nf) {
    a.NF *= 2;
    ++a.logNF;
  }
  const int W = 2 * a.NF;
  a.G = (a.ppp + a.NF - 1) / a.NF;
  a.g0 = 0;
  if (k.line1 > k.line0) {  // a sub-range of line blocks
    if (k.line0 % W || (k.line1 % W && k.line1 != a.nrow)) return HFB_ERR_ARGUMENT;
    a.g0 = k.line0 / W;
    a.G = (k.line1 + W - 1) / W - a.g0;
  }
  a.max_per_sm = k.max_per_sm;
  a.rowslot = ((a.N + 4) + 1) & ~1;
  int gb = std::max(2 * a.rowslot, 2 * G::BUF);
  // tensor-store outputs: rows stored whole (position N lands in the row's
  // padding, so ld >= M), 16-byte aligned rows and planes
  a.flags = k.flags;
  a.wc = k.wc;
  a.desc = k.mode == kYB;
  a.dbg = g_tune_wave_dbg;
  // packed output: the line's M positions as pack_parts pieces of pack_kp in the
  // exchange blocks (whole 128-byte segments per piece)
  a.packed = k.pack_parts > 0;
  if (a.packed && ((k.mode != kRow && k.mode != kTload) || k.pack_kp % 16 ||
                   (long long)k.pack_kp * k.pack_parts != M || (k.pack_bstride & 1) ||
                   (reinterpret_cast<uintptr_t>(a.dst) & 15) || k.pack_parts > 256))
    return HFB_ERR_ARGUMENT;
  a.tstore = a.packed ||
             ((k.mode != kTran && k.mode != kYF2) &&
              (g_tune_tstore || k.mode == kYF || k.mode == kYB) && M >= 16 &&
              a.out_ld >= M && !(reinterpret_cast<uintptr_t>(a.dst) & 15) && !(a.out_ld & 1) &&
              !(a.out_ps & 1));
  if ((k.mode == kYF || k.mode == kYB) && !a.tstore) return HFB_ERR_ARGUMENT;
  a.pbulk = !a.tstore && (k.mode == kRow || k.mode == kTload) && E == 16 && g_tune_pbulk &&
            a.out_ld == a.N && !(reinterpret_cast<uintptr_t>(a.dst) & 7);
  // (measured: 4.47 -> 4.22 ms at M = 1024, 46.3 -> 45.3 ms at M = 2048, slower at 512)
  a.ustore = !a.tstore && !a.pbulk && (k.mode == kRow || k.mode == kTload) && E == 16 &&
             g_tune_ustore && (M == 1024 || M == 2048) && a.out_ld == a.N &&
             !(reinterpret_cast<uintptr_t>(a.dst) & 15);
  // spare KB + rows -1 .. 2N/16 + 1 of the flat box
  if (a.ustore) gb = std::max(gb, 128 + ((2 * a.N) / 16 + 3) * 16);
  if (a.tstore || a.ustore) {
    gb = (gb + 127) & ~127;  // every group box 1-KB aligned (128B swizzle atoms)
  } else if (T >= 32) {
    gb = (gb + 31) & ~31;  // 256-byte aligned group buffers (the engine's XOR byte addresses)
  } else {
    const int want = 16 / a.NF;  // group offsets spread over the 8 16-byte bank groups
    while (gb % 16 != want % 16) ++gb;
  }
  a.gbuf = gb;
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  if (a.packed) {
    auto enc = tensor_encoder();
    if (!enc) return HFB_ERR_CUDA;
    const cuuint64_t kp = (cuuint64_t)k.pack_kp;
    cuuint64_t dims[5] = {16, kp / 16, (cuuint64_t)k.pack_parts, (cuuint64_t)a.nrow,
                          (cuuint64_t)(a.z0 + a.nz)};
    cuuint64_t strides[4] = {128, (cuuint64_t)k.pack_bstride * 8, kp * 8,
                             (cuuint64_t)a.nrow * kp * 8};
    cuuint32_t box[5] = {16, (cuuint32_t)(kp / 16), (cuuint32_t)k.pack_parts, 2, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a.dst, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HFB_ERR_ARGUMENT;
  } else if (a.tstore) {
    auto enc = tensor_encoder();
    if (!enc) return HFB_ERR_CUDA;
    cuuint64_t dims[4] = {16, (cuuint64_t)(M / 16), (cuuint64_t)a.nrow,
                          (cuuint64_t)(a.z0 + a.nz)};
    cuuint64_t strides[3] = {128, (cuuint64_t)a.out_ld * 8, (cuuint64_t)a.out_ps * 8};
    cuuint32_t box[4] = {16, (cuuint32_t)(M / 16), 2, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a.dst, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HFB_ERR_ARGUMENT;
  }
  // decoupled groups: row passes, and column passes at M = 2048 (measured: x 3.90 -> 3.78,
  // inverse y 3.92 -> 3.82 ms at 1023^3; final x-pass 46.3 -> 42.3 ms at 2047^3; the
  // column passes at M = 1024 got slower with per-group boxes, 4.28 -> 4.57 ms)
  // late prefetch (key 29: 1 all passes, 2 the flat-row-store passes only).
  // Measured at 1023^3 (same box): final pass 4.87 -> 4.62 ms, the other
  // passes 0.05-0.12 ms slower.
  // After the engine's address-generation work the M = 2048 final pass is
  // faster with the early prefetch again (47.0 -> 38.9 ms at 2047^3, same box),
  // the M = 1024 one still with the late one (3.97 vs 4.11 ms): key 29 = 2 now
  // means the M = 1024 flat-row-store passes only.
  a.late = tuning(29) == 1 || (tuning(29) == 2 && a.ustore && M == 1024);
  // key 14 = 2: also decouple the groups of the M = 1024 column pass that stores
  // into the user's array (flat-row stores; the final inverse-x pass)
  a.indep = (k.mode == kRow || k.mode == kYB || (k.mode == kTload && M == 2048) ||
             (k.mode == kTload && a.ustore && g_tune_indep == 2)) &&
            (a.tstore || a.ustore) && (g_tune_indep || k.mode == kYB) && T >= 32;
  if (k.mode == kYB && !a.indep) return HFB_ERR_ARGUMENT;
  CUtensorMap umap;
  memset(&umap, 0, sizeof(umap));
  if (a.ustore) {
    // the destination as flat 128-byte rows: [16 doubles][rows], boxes of the two possible
    // full-row counts of a line-pair run (2N/16 and one less)
    auto enc = tensor_encoder();
    if (!enc) return HFB_ERR_CUDA;
    const long long total = (long long)(a.z0 + a.nz) * a.out_ps;  // doubles from dst
    cuuint64_t dims[2] = {16, (cuuint64_t)(total / 16)};
    cuuint64_t strides[1] = {128};
    cuuint32_t estr[2] = {1, 1};
    for (int h = 0; h < 2; ++h) {
      cuuint32_t box[2] = {16, (cuuint32_t)((2 * a.N) / 16 - h)};
      CUresult r = enc(h ? &omap : &umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.dst, dims, strides,
                       box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return HFB_ERR_ARGUMENT;
    }
  }
  long long stage = (long long)a.NF * a.gbuf;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (k.mode == kTload || k.mode == kYF || k.mode == kYF2) {
    a.boxn = std::min(256, M);
    a.nbox = M / a.boxn;
    stage = std::max<long long>(stage, (long long)a.nbox * a.boxn * W);
    auto enc = tensor_encoder();
    if (!enc) return HFB_ERR_CUDA;
    if ((reinterpret_cast<uintptr_t>(a.src) & 15) || (a.in_ld & 1) || (a.in_ps & 1))
      return HFB_ERR_ARGUMENT;
    cuuint64_t dims[3] = {(cuuint64_t)a.nrow, (cuuint64_t)a.N, (cuuint64_t)(a.z0 + a.nz)};
    cuuint64_t strides[2] = {(cuuint64_t)a.in_ld * 8, (cuuint64_t)a.in_ps * 8};
    // indep: one unswizzled [pos][2 lines] box per group
    cuuint32_t box[3] = {(cuuint32_t)(a.indep ? 2 : W), (cuuint32_t)a.boxn, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.src), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     a.indep     ? CU_TENSOR_MAP_SWIZZLE_NONE
                     : a.NF == 8 ? CU_TENSOR_MAP_SWIZZLE_128B
                     : a.NF == 4 ? CU_TENSOR_MAP_SWIZZLE_64B
                     : a.NF == 2 ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : CU_TENSOR_MAP_SWIZZLE_NONE,
                     g_tune_l2 == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                     : g_tune_l2 == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                     : g_tune_l2 == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                      : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HFB_ERR_ARGUMENT;
  }
  a.stage = (int)((stage + 127) & ~127LL);
  a.vec_out = (k.mode == kTran) && !(reinterpret_cast<uintptr_t>(a.dst) & 15) &&
              !(a.out_ld & 1) && !(a.out_ps & 1);
  const int threads = a.NF * T;
  size_t sm = 1024 + (size_t)2 * a.stage * sizeof(double) +
              (threads / 32 + 1) * sizeof(double2) + 2 * sizeof(uint64_t);
  if (k.mode == kYF) {
    sm += sizeof(double) * ((size_t)2 * a.NF * M + M);  // c carry + permuted cy
    a.coef = k.coef;
    a.cx = k.cx;
    a.cy = k.cy;
    a.thr = k.thr;
    a.err = k.err;
    a.ck = k.cp;
    a.ck_ld = a.out_ld;
    a.ck_ps = a.out_ps;
    a.nz_total = k.nz_total;
    a.ny_total = a.N;
    a.nx_total = a.nrow;
    return launch_stream<P, E, kYF>(a, c, tmap, omap, umap, threads, sm, st);
  }
  if (k.mode == kYF2 || k.mode == kYB) {
    a.coef = k.coef;
    a.cx = k.cx;
    a.cy = k.cy;
    a.thr = k.thr;
    a.err = k.err;
    a.ck = k.cp;  // the full cp volume, layout of the y-pass output rows
    // (n, m) rows of the mode volume: the kYF2 output / the kYB input layout
    a.ck_ld = k.mode == kYF2 ? a.out_ld : a.in_ld;
    a.ck_ps = k.mode == kYF2 ? a.out_ps : a.in_ps;
    a.nz_total = k.nz_total;
    a.ny_total = a.N;
    a.nx_total = a.nrow;
    if constexpr (P <= 10 && E == 16) {
      if (k.mode == kYF2) return launch_stream<P, E, kYF2>(a, c, tmap, omap, umap, threads, sm, st);
      return launch_stream<P, E, kYB>(a, c, tmap, omap, umap, threads, sm, st);
    }
    return HFB_ERR_ARGUMENT;
  }
  if (k.mode == kTran) return launch_stream<P, E, kTran>(a, c, tmap, omap, umap, threads, sm, st);
  if (k.mode == kTload) return launch_stream<P, E, kTload>(a, c, tmap, omap, umap, threads, sm, st);
  if (k.split_parts > 0) {
    // input lines split over exchange blocks: whole 16-byte aligned pieces
    if ((long long)k.split_kp * k.split_parts != M || (k.split_kp & 1) || (k.split_bstride & 1) ||
        (reinterpret_cast<uintptr_t>(a.src) & 15))
      return HFB_ERR_ARGUMENT;
    a.sp_parts = k.split_parts;
    a.sp_kp = k.split_kp;
    a.sp_bstride = k.split_bstride;
    if constexpr (E == 16 && P >= 6)
      return launch_stream<P, E, kRowS>(a, c, tmap, omap, umap, threads, sm, st);
    return HFB_ERR_ARGUMENT;
  }
  return launch_stream<P, E, kRow>(a, c, tmap, omap, umap, threads, sm, st);
}

template <int P>
static int launch_p(const Dst16Call& k, StreamArgs a, const FftArgs& c, cudaStream_t st) {
  // E = 32 on request, and whenever E = 16 would need more than 128 threads
  // per line pair (M = 4096)
  if constexpr (P >= 12) {
    return launch_pe<P, 32>(k, a, c, st);
  } else if constexpr (P >= 5) {
    if (g_tune_E == 32) return launch_pe<P, 32>(k, a, c, st);
  }
  return launch_pe<P, 16>(k, a, c, st);
}

int tuning(int key) {
  switch (key) {
    case 0: return g_tune_E;
    case 1: return g_tune_NF;
    case 2: return g_tune_l2;
    case 3: return g_tune_order;
    case 4: return g_tune_tstore;
    case 5: return g_tune_fuse;
    case 6: return g_tune_overlap;
    case 9: return g_tune_pbulk;
    case 7: return g_tune_cap_dst;
    case 8: return g_tune_cap_th;
    case 10: return g_tune_cap_all;
    case 11: return g_tune_carry_ms;
    case 12: return g_tune_carry_cap;
    case 13: return g_tune_ustore;
    case 14: return g_tune_indep;
    case 16: return g_tune_dmma;
    case 17: return g_tune_dense_max;
    case 18: return g_tune_dmma2d;
    case 19: return g_tune_thomas_smem;
    case 20: return g_tune_rhs_march;
    case 21: return g_tune_wave;
    case 22: return g_tune_wave_dbg;
    case 23: return g_tune_xsparse;
    case 24: return g_tune_s27;
    case 25: return g_tune_s27_rj;
    case 26: return g_tune_thomas_stages;
    case 27: return g_tune_s27_tile;
    case 28: return g_tune_thomas_narrow;
    case 29: return g_tune_late;
    case 30: return g_tune_thomas_kc;
    case 31: return g_tune_zinv;
    case 32: return g_tune_ckcache;
    default: return 0;
  }
}

void set_tuning(int key, int value) {
  if (key == 0) g_tune_E = (value == 32) ? 32 : 16;
  if (key == 1) g_tune_NF = value;
  if (key == 2) g_tune_l2 = value;
  if (key == 3) g_tune_order = value;
  if (key == 4) g_tune_tstore = value ? 1 : 0;
  if (key == 5) g_tune_fuse = value ? 1 : 0;
  if (key == 6) g_tune_overlap = value ? 1 : 0;
  if (key == 9) g_tune_pbulk = value ? 1 : 0;
  if (key == 7) g_tune_cap_dst = value;
  if (key == 8) g_tune_cap_th = value;
  if (key == 10) g_tune_cap_all = value;
  if (key == 11) g_tune_carry_ms = value;
  if (key == 12) g_tune_carry_cap = value;
  if (key == 13) g_tune_ustore = value ? 1 : 0;
  if (key == 14) g_tune_indep = value;
  if (key == 16) g_tune_dmma = value ? 1 : 0;
  if (key == 17) g_tune_dense_max = value;
  if (key == 18) g_tune_dmma2d = value;
  if (key == 19) g_tune_thomas_smem = value ? 1 : 0;
  if (key == 20) g_tune_rhs_march = value;
  if (key == 21) g_tune_wave = value ? 1 : 0;
  if (key == 22) g_tune_wave_dbg = value;
  if (key == 23) g_tune_xsparse = value ? 1 : 0;
  if (key == 24) g_tune_s27 = value;
  if (key == 25) g_tune_s27_rj = value;
  if (key == 26) g_tune_thomas_stages = value;
  if (key == 27) g_tune_s27_tile = value ? 1 : 0;
  if (key == 28) g_tune_thomas_narrow = value;
  if (key == 29) g_tune_late = value;
  if (key == 30) g_tune_thomas_kc = value;
  if (key == 31) g_tune_zinv = value ? 1 : 0;
  if (key == 32) g_tune_ckcache = value ? 1 : 0;
}

int launch_dst16_mode(const Dst16Call& k, cudaStream_t st) {
  if (k.nz <= 0 || k.nrow <= 0) return HFB_OK;
  if (k.mode < kRow || k.mode > kYB) return HFB_ERR_ARGUMENT;
  if (k.mode == kYF && (k.z0 != 0 || !k.coef || !k.cp)) return HFB_ERR_ARGUMENT;
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
