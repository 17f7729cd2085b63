// Streaming Thomas sweep for the transposed, padded (l, n, m) layout of the
// one-call solve: kernel (c) fed by the TMA engine.
//
// A CTA owns a contiguous block of BM = 256 modes (one row segment: fixed x-mode
// n, y-modes m0..m0+255) and walks the levels in chunks of K = 8. Every chunk's
// 8 rows (and the chunk's 8 x 12 stencil weights) arrive by 1D bulk copies into
// a 3-stage shared-memory ring, two chunks ahead of the compute; results leave
// by 1D bulk stores. The memory-level parallelism therefore comes from the
// copy engine (~32 KB in flight per CTA), not from thread occupancy, which is
// what the plain thread-per-mode sweep lacks (its per-level loads sit inside
// the recurrence's latency chain).
//
// Arithmetic is the same as thomas.cu (bitwise): cp is kept only at the last
// level of each chunk (cpk, one plane per chunk) and recomputed per chunk in
// the back substitution, 34 B/point of HBM traffic instead of 48.
#include "hfb_internal.cuh"
#include "tma.cuh"

namespace hfb {

namespace {
constexpr int BMAX = 256;  // modes per CTA block = threads (128 for narrow y-slabs)
constexpr int K = kThomasChunk;  // levels per chunk

struct TmaArgs {
  double* w;           // data (l, n, m): x' / W in place
  double* cpk;         // checkpoints: plane q holds cp at level q*K + K - 1
  const double* coef;  // [l][k][(4a, 2b, 2c, d)]
  const double* pq;    // [n][l][k][(P, Q)] (eig_pq), the per-level path's weights
  const double* cx;
  const double* cy;
  int nz, nrows, ncols, nbpr;  // levels, rows (n), cols (m), blocks per row
  long long ld, ps;            // row / plane strides (doubles), ld even
  double thr;
  unsigned long long* err;
  int nx, ny_total;
  int bwd_only;  // forward sweep already done (x' and checkpoints in place)
  int m_off;     // global y-mode of column 0 (a y-slab of modes)
  int row0;      // first row (x-mode) of this launch
  const int* lvl;  // level -> plane of the data (null: identity), e.g. a chunked y-slab
  int xsparse;     // forward stores x' only at each chunk's first level (see below)
  int ck_ro;       // cpk already holds this matrix's checkpoints: the forward stores none
};

__device__ __forceinline__ double eig_s(const double* co, double cx, double cy, double cxy) {
  (void)cxy;
  return eig_pq(co, cx, cy);
}
}  // namespace

// KC levels per chunk (tuning key 30; 16 halves the chunk barriers and the
// checkpoint traffic, at twice the shared memory per stage).
//
// ZI: the weight table is the same on every level (a z-invariant operator, e.g.
// constant k or the constant-coefficient convection-diffusion of cfg4; flagged
// by hfb_plan_set_coefficients, tuning key 31). The three eigenvalues of each
// mode are then computed once per block, with the same expressions (so the same
// bits), and the chunks carry no weights.
// (P, Q) table: one thread per (n, l, k); the same fma's as eig_pq
__global__ void pq_kernel(const double* __restrict__ coef, const double* __restrict__ cx,
                          double* __restrict__ pq, int nx, int nz) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)nx * nz * 3) return;
  const int k = (int)(e % 3);
  const long long l = (e / 3) % nz, n = e / (3LL * nz);
  const double* co = coef + l * 12 + 4 * k;
  const double c = __ldg(cx + n);
  pq[2 * e] = eig_p(co[0], co[2], c);
  pq[2 * e + 1] = eig_q(co[1], co[3], c);
}

int build_pq(hfb_plan* p) {
  const long long n = (long long)p->nx * p->nz * 3;
  if (!p->pq) HFB_CUDA(cudaMalloc(&p->pq, sizeof(double) * 2 * n));
  pq_kernel<<<(unsigned)((n + 255) / 256), 256>>>(p->coef, p->cx, p->pq, p->nx, p->nz);
  HFB_LAUNCHED();
  HFB_CUDA(cudaDeviceSynchronize());  // the table is complete before any solve reads it
  return HFB_OK;
}

template <int BM, int S, int KC, bool ZI>
__global__ void __launch_bounds__(BM) thomas_tma_kernel(TmaArgs a) {
  constexpr int K = KC;
  extern __shared__ __align__(16) double dyn[];
  double(*sdat)[K][BM] = reinterpret_cast<double(*)[K][BM]>(dyn);
  double(*scoef)[K * 12] = reinterpret_cast<double(*)[K * 12]>(dyn + S * K * BM);
  __shared__ uint64_t bar[S];
  const int tid = threadIdx.x;
  const int nchunk = (a.nz + K - 1) / K;
  const int ntask = 2 * nchunk;  // forward chunks ascending, then backward descending
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of stage s

  for (long long blk = blockIdx.x; blk < (long long)a.nrows * a.nbpr; blk += gridDim.x) {
    const int n = a.row0 + (int)(blk / a.nbpr);
    const int m0 = (int)(blk % a.nbpr) * BM;
    const int cols = min(BM, a.ncols - m0);
    const uint32_t rowbytes = (uint32_t)(((cols + 1) & ~1) * 8);  // ld is even
    double* base = a.w + (long long)n * a.ld + m0;
    auto chunk_of = [&](int task) { return task < nchunk ? task : ntask - 1 - task; };
    auto plane_of = [&](int l) -> long long { return a.lvl ? __ldg(a.lvl + l) : l; };
    // thread 0: bring chunk `task` into stage s
    auto issue = [&](int task, int s) {
      const int c = chunk_of(task);
      const int l0 = c * K, nl = min(K, a.nz - l0);
      mbar_arrive_expect_tx(&bar[s], nl * rowbytes + (ZI ? 0u : (uint32_t)(nl * 6 * 8)));
      for (int i = 0; i < nl; ++i)
        bulk_g2s(&sdat[s][i][0], base + plane_of(l0 + i) * a.ps, rowbytes, &bar[s]);
      if (!ZI)
        bulk_g2s(&scoef[s][0], a.pq + ((long long)n * a.nz + l0) * 6, (uint32_t)(nl * 6 * 8),
                 &bar[s]);
    };
    const bool live = tid < cols;
    const int m = m0 + tid;
    const double cxv = __ldg(a.cx + n);
    const double cyv = live ? __ldg(a.cy + a.m_off + m) : 0.0;
    const double cxy = cxv * cyv;
    double* ck = a.cpk + (long long)n * a.ld + m0 + tid;
    double zl = 0.0, zd = 0.0, zu = 0.0;
    if constexpr (ZI) {
      zl = eig_s(a.coef, cxv, cyv, cxy);
      zd = eig_s(a.coef + 4, cxv, cyv, cxy);
      zu = eig_s(a.coef + 8, cxv, cyv, cxy);
    }

    // The last forward chunk stays in its stage and is the first backward chunk
    // (no store, no reload), so stages run task % S forward and (task-1) % S
    // backward.
    // backward-only: tasks nchunk .. 2 nchunk - 1, every chunk loaded
    const int task0 = a.bwd_only ? nchunk : 0;
    auto stage_of = [&](int task) {
      return a.bwd_only ? (task - task0) % S : task < nchunk ? task % S : (task - 1) % S;
    };
    auto needs_load = [&](int task) { return a.bwd_only || task != nchunk; };
    // prefetch distance in tasks: 2 (1 with two stages). The stage that task
    // t + D fills was last used by task t + D - S: task t - 1 with 3 (or 2)
    // stages, whose store is the last one committed; task t - 2 with 4.
    constexpr int D = S >= 3 ? 2 : 1;
    if (tid == 0)
      for (int q = 0; q < D; ++q)
        if (task0 + q < ntask && needs_load(task0 + q)) issue(task0 + q, stage_of(task0 + q));
    // Sparse x' (tuning key 23, not with bwd_only): the forward sweep stores x'
    // only at level l0 of every chunk (levels l0+1 .. l0+K-1 keep F-hat in
    // place), and the back substitution recomputes x'_l = (F_l - lo x'_{l-1}) rr_l
    // inside the cp recomputation it runs anyway, bit for bit the forward's
    // expression: 27 instead of 34 B/point of HBM traffic, no extra registers
    // (the recomputed values go back into the staged chunk). The last forward
    // chunk stays on chip with every x' as before.
    const bool xs = a.xsparse && !a.bwd_only;
    double c = 0.0, x = 0.0, cknext = 0.0;
    if (a.bwd_only && live && nchunk > 1) cknext = ck[(long long)(nchunk - 2) * a.ps];
    for (int task = task0; task < ntask; ++task) {
      const int s = stage_of(task);
      if (tid == 0 && task + D < ntask && needs_load(task + D)) {
        // backward reloads must see the forward stores; otherwise only the
        // stage's previous store has to be done reading shared memory
        // The stage's previous user must have been read out by its store.
        // With 3 stages that store is the one issued at the end of the last
        // task; with 4 it is the store before that.
        if constexpr (S >= 4) bulk_wait_read<1>(); else bulk_wait_read<0>();
        if (!a.bwd_only && task + D > nchunk) {
          // a backward reload needs its chunk's forward store complete in
          // global memory; the store groups committed after it (one per task
          // but nchunk - 1, the last at the end of task - 1) may be in flight
          const int cc = ntask - 1 - (task + D);
          const int after =
              (task - 1 - cc) - ((cc < nchunk - 1 && nchunk - 1 <= task - 1) ? 1 : 0);
          bulk_wait_upto(after);
        }
        fence_proxy_async_smem();
        issue(task + D, stage_of(task + D));
      }
      if (needs_load(task)) {
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
      }
      const int cidx = chunk_of(task);
      const int l0 = cidx * K, nl = min(K, a.nz - l0);
      const double* co = &scoef[s][0];
      // the level's (lower, diagonal, upper) eigenvalues of this mode
      // (the chunk carries the block's x-mode's (P, Q) pairs: one fma each)
      auto EL = [&](int i) { return ZI ? zl : fma(co[i * 6], cyv, co[i * 6 + 1]); };
      auto ED = [&](int i) { return ZI ? zd : fma(co[i * 6 + 2], cyv, co[i * 6 + 3]); };
      auto EU = [&](int i) { return ZI ? zu : fma(co[i * 6 + 4], cyv, co[i * 6 + 5]); };
      // Interior chunks (all K levels present, not level 0, below the top
      // level) run a copy of the loops without the per-level guards, and note
      // a vanishing pivot as the chunk's first failing level (one select per
      // level instead of a branch); the arithmetic is the guarded loop's.
      const bool inner = nl == K && l0 > 0 && l0 + K < a.nz;
      if (task < nchunk) {
        // forward elimination over levels l0 .. l0 + nl - 1
        const bool keep_all = !xs || task == nchunk - 1;
        if (inner) {
          int bad = K;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const double lo = EL(i);
            const double di = ED(i);
            const double up = EU(i);
            const double den = fma(-lo, c, di);
            bad = (fabs(den) < a.thr && bad == K) ? i : bad;
            const double rr = rcp_fast(den);
            x = fma(-lo, x, sdat[s][i][tid]) * rr;
            if (keep_all || i == 0) sdat[s][i][tid] = x;
            c = up * rr;
          }
          if (live && !a.ck_ro) ck[(long long)cidx * a.ps] = c;
          if (live && bad < K) {
            const unsigned long long key =
                ((unsigned long long)(l0 + bad) * (unsigned long long)a.ny_total +
                 (unsigned long long)(a.m_off + m)) *
                    (unsigned long long)a.nx +
                (unsigned long long)n;
            atomicMin(a.err, key);
          }
        } else {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            if (i < nl) {
              const int l = l0 + i;
              const double lo = EL(i);
              const double di = ED(i);
              const double up = EU(i);
              const double den = (l == 0) ? di : fma(-lo, c, di);
              if (live && fabs(den) < a.thr) {
                const unsigned long long key =
                    ((unsigned long long)l * (unsigned long long)a.ny_total +
                     (unsigned long long)(a.m_off + m)) *
                        (unsigned long long)a.nx +
                    (unsigned long long)n;
                atomicMin(a.err, key);
              }
              const double rr = rcp_fast(den);
              x = ((l == 0) ? sdat[s][i][tid] : fma(-lo, x, sdat[s][i][tid])) * rr;
              if (keep_all || i == 0) sdat[s][i][tid] = x;
              if (l < a.nz - 1) {
                c = up * rr;
                if (i == K - 1 && live && !a.ck_ro) ck[(long long)cidx * a.ps] = c;
              }
            }
          }
        }
        if (live && task == nchunk - 1 && nchunk > 1) cknext = ck[(long long)(nchunk - 2) * a.ps];
      } else {
        // back substitution over levels l0 + nl - 1 .. l0 (x holds W at the level above)
        if (a.bwd_only && task == task0) x = sdat[s][nl - 1][tid];  // W = x' at the top
        double cprev = cknext;
        if (cidx >= 2 && live) cknext = ck[(long long)(cidx - 2) * a.ps];
        double cb[K];
        // x' of this chunk to recompute (every chunk but the on-chip last one)
        const bool rec = xs && task != nchunk;
        double xr = rec ? sdat[s][0][tid] : 0.0;
        if (inner) {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const double di = ED(i);
            const double lo = EL(i);
            const double rr = rcp_fast(fma(-lo, cprev, di));
            if (rec && i > 0) {
              xr = fma(-lo, xr, sdat[s][i][tid]) * rr;
              sdat[s][i][tid] = xr;
            }
            cprev = EU(i) * rr;
            cb[i] = cprev;
          }
#pragma unroll
          for (int i = K - 1; i >= 0; --i) {
            x = fma(-cb[i], x, sdat[s][i][tid]);
            sdat[s][i][tid] = x;
          }
        } else {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const int l = l0 + i;
            if (i < nl && l < a.nz - 1) {
              const double di = ED(i);
              const double lo = EL(i);
              const double dl = (l == 0) ? di : fma(-lo, cprev, di);
              const double rr = rcp_fast(dl);
              if (rec && i > 0) {
                xr = fma(-lo, xr, sdat[s][i][tid]) * rr;
                sdat[s][i][tid] = xr;
              }
              cprev = EU(i) * rr;
              cb[i] = cprev;
            }
          }
#pragma unroll
          for (int i = K - 1; i >= 0; --i) {
            const int l = l0 + i;
            if (i < nl && l < a.nz - 1) {
              x = fma(-cb[i], x, sdat[s][i][tid]);
              sdat[s][i][tid] = x;
            }
          }
        }
      }
      __syncthreads();  // every thread's results for this chunk are in sdat[s]
      if (tid == 0 && task != nchunk - 1) {
        fence_proxy_async_smem();
        const int nst = (xs && task < nchunk) ? 1 : nl;  // sparse x': level l0 only
        for (int i = 0; i < nst; ++i)
          bulk_s2g(base + plane_of(l0 + i) * a.ps, &sdat[s][i][0], rowbytes);
        bulk_commit();
      }
    }
    if (tid == 0) bulk_wait<0>();  // stores done before the stages are refilled
    __syncthreads();
  }
}

// Small systems (n_z <= 256, e.g. cfg1 / cfg2): one warp owns 32 modes of a row
// and holds all their levels in shared memory (data and cp, 512 n_z bytes), so
// the sweeps run without a copy ring or per-chunk barriers: load every level,
// eliminate up, substitute down, store every level. Latency-bound problems
// (a few thousand modes, a 2 n_z-step recurrence each) are what it is for. The
// arithmetic is thomas_tma_kernel's expression for expression (cp is kept
// instead of recomputed: the same values), so results are bitwise the same.
__global__ void __launch_bounds__(32) thomas_smem_kernel(TmaArgs a) {
  extern __shared__ __align__(16) double smq[];
  double* sd = smq;                    // [nz][32] data
  double* sc = sd + (long long)a.nz * 32;   // [nz][32] cp
  double* co = sc + (long long)a.nz * 32;   // [nz][12] weights
  const int t = threadIdx.x;
  for (int e = t; e < a.nz * 12; e += 32) co[e] = __ldg(a.coef + e);
  const long long blk = blockIdx.x;
  const int n = a.row0 + (int)(blk / a.nbpr);
  const int m0 = (int)(blk % a.nbpr) * 32;
  const int cols = min(32, a.ncols - m0);
  const bool live = t < cols;
  const int m = m0 + t;
  double* base = a.w + (long long)n * a.ld + m0 + t;
  if (live) {  // 16 independent loads in flight per thread
    int l = 0;
    for (; l + 16 <= a.nz; l += 16) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = base[(long long)(l + q) * a.ps];
#pragma unroll
      for (int q = 0; q < 16; ++q) sd[(l + q) * 32 + t] = v[q];
    }
    for (; l < a.nz; ++l) sd[l * 32 + t] = base[(long long)l * a.ps];
  }
  __syncwarp();
  const double cxv = __ldg(a.cx + n);
  const double cyv = live ? __ldg(a.cy + a.m_off + m) : 0.0;
  const double cxy = cxv * cyv;
  double c = 0.0, x = 0.0;
  for (int l = 0; l < a.nz; ++l) {
    const double* cl = co + l * 12;
    const double lo = eig_s(cl, cxv, cyv, cxy);
    const double di = eig_s(cl + 4, cxv, cyv, cxy);
    const double up = eig_s(cl + 8, cxv, cyv, cxy);
    const double den = (l == 0) ? di : fma(-lo, c, di);
    if (live && fabs(den) < a.thr) {
      const unsigned long long key =
          ((unsigned long long)l * (unsigned long long)a.ny_total +
           (unsigned long long)(a.m_off + m)) *
              (unsigned long long)a.nx +
          (unsigned long long)n;
      atomicMin(a.err, key);
    }
    const double rr = rcp_fast(den);
    x = ((l == 0) ? sd[l * 32 + t] : fma(-lo, x, sd[l * 32 + t])) * rr;
    sd[l * 32 + t] = x;
    if (l < a.nz - 1) {
      c = up * rr;
      sc[l * 32 + t] = c;
    }
  }
  for (int l = a.nz - 2; l >= 0; --l) {
    x = fma(-sc[l * 32 + t], x, sd[l * 32 + t]);
    sd[l * 32 + t] = x;
  }
  if (live)
    for (int l = 0; l < a.nz; ++l) base[(long long)l * a.ps] = sd[l * 32 + t];
}

int launch_thomas_tma_cached(hfb_plan* p, double* data, double* cpk, long long ld, long long ps,
                             cudaStream_t st) {
  if (!tuning(32) || p->nz <= 256) return launch_thomas_tma(p, data, cpk, ld, ps, st, 0);
  // what the cached checkpoints depend on: the coefficients, the layout and the
  // chunk length
  const unsigned long long sig = (p->coef_epoch << 20) ^ ((unsigned long long)ld << 44) ^
                                 ((unsigned long long)ps * 0x9E3779B97F4A7C15ull) ^
                                 (unsigned long long)(tuning(30) ? 16 : K);
  const int kc = tuning(30) ? 16 : K;
  const size_t need = sizeof(double) * (size_t)((p->nz + kc - 1) / kc) * (size_t)ps;
  if (!p->ck_cache || p->ck_cache_bytes < need) {
    if (p->ck_cache) cudaFree(p->ck_cache);
    p->ck_cache = nullptr;
    p->ck_cache_bytes = 0;
    p->ck_valid = 0;
    if (cudaMalloc(&p->ck_cache, need) == cudaSuccess) {
      p->ck_cache_bytes = need;
    } else {
      (void)cudaGetLastError();  // no room: solve with the workspace's checkpoints
      p->ck_cache = nullptr;
    }
  }
  if (!p->ck_cache) return launch_thomas_tma(p, data, cpk, ld, ps, st, 0);
  const int ro = p->ck_valid && p->ck_sig == sig && p->ck_stream == st;
  const int rc = launch_thomas_tma(p, data, p->ck_cache, ld, ps, st, 0, ro);
  if (rc == HFB_OK && !ro) {
    p->ck_valid = 1;
    p->ck_sig = sig;
    p->ck_stream = st;
  }
  return rc;
}

int launch_thomas_tma(hfb_plan* p, double* data, double* cpk, long long ld, long long ps,
                      cudaStream_t st, int bwd_only, int ck_ro) {
  // the whole column on chip (tuning key 19, default on) when the modes fit in
  // a few waves of it; many modes keep the bandwidth-bound copy ring
  const size_t sm_small = sizeof(double) * ((size_t)p->nz * 64 + (size_t)p->nz * 12);
  int per_sm_small = 0, sms_small = 148, dev_small = 0;
  if (!bwd_only && p->nz <= 256 && tuning(19)) {
    HFB_CUDA(cudaFuncSetAttribute(thomas_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm_small));
    HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_small, thomas_smem_kernel, 32,
                                                           sm_small));
    if (cudaGetDevice(&dev_small) == cudaSuccess)
      cudaDeviceGetAttribute(&sms_small, cudaDevAttrMultiProcessorCount, dev_small);
  }
  const long long blocks_small = (long long)p->nx * ((p->ny + 31) / 32);
  if (per_sm_small > 0 && blocks_small <= 4LL * sms_small * per_sm_small) {
    TmaArgs a = {};
    a.w = data;
    a.coef = p->coef;
    a.cx = p->cx;
    a.cy = p->cy;
    a.nz = p->nz;
    a.nrows = p->nx;
    a.ncols = p->ny;
    a.nbpr = (p->ny + 31) / 32;
    a.ld = ld;
    a.ps = ps;
    a.thr = p->thr;
    a.err = p->err;
    a.nx = p->nx;
    a.ny_total = p->ny;
    thomas_smem_kernel<<<(unsigned)blocks_small, 32, sm_small, st>>>(a);
    HFB_LAUNCHED();
    return HFB_OK;
  }
  return launch_thomas_tma_cols(p, data, cpk, ld, ps, p->ny, 0, st, bwd_only, 0, -1, 0, nullptr,
                                ck_ro);
}

int launch_thomas_tma_cols(hfb_plan* p, double* data, double* cpk, long long ld, long long ps,
                           int ncols, int m_off, cudaStream_t st, int bwd_only, int row0,
                           int row1, int max_per_sm, const int* lvl, int ck_ro) {
  if (row1 < 0) row1 = p->nx;
  if (p->nz < 1 || ncols < 1 || row1 <= row0) return HFB_OK;
  TmaArgs a;
  a.bwd_only = bwd_only;
  a.m_off = m_off;
  a.row0 = row0;
  a.lvl = lvl;
  a.xsparse = tuning(23);
  a.ck_ro = ck_ro && !bwd_only;
  a.w = data;
  a.cpk = cpk;
  a.coef = p->coef;
  a.pq = p->pq;
  a.cx = p->cx;
  a.cy = p->cy;
  a.nz = p->nz;
  a.nrows = row1 - row0;
  a.ncols = ncols;
  // narrow y-slabs (multi-GPU, P >= 8) would leave half of a 256-mode block idle
  // (tuning key 28 = 1: 128-mode blocks everywhere — 4-warp barriers, more CTAs)
  const int BM = (ncols <= 128 || tuning(28) == 1) ? 128 : BMAX;
  a.nbpr = (ncols + BM - 1) / BM;
  a.ld = ld;
  a.ps = ps;
  a.thr = p->thr;
  a.err = p->err;
  a.nx = p->nx;
  a.ny_total = p->ny;
  // ring stages (tuning key 26: 3 or 4; 4 lets the refill skip waiting for the
  // store issued just before, at 16 KB more shared memory per 256-mode CTA)
  const int S = (bwd_only || tuning(26) != 4) ? 3 : 4;
  // chunk shape (tuning key 30, one-call and mode-slab paths; bwd_only keeps the
  // 8-level checkpoints its producers wrote): 1 = 16 levels, 3 stages;
  // 2 = 16 levels, 2 stages
  const int kc = bwd_only ? 0 : tuning(30);
  const int KC = kc ? 16 : K, SS = kc == 2 ? 2 : S;
  const size_t sm = sizeof(double) * (size_t)SS * (KC * BM + KC * 12);
  // z-invariant weights (key 31): eigenvalues once per mode block
  const bool zi = p->zinv && tuning(31);
  decltype(&thomas_tma_kernel<BMAX, 3, K, false>) kern;
  if (zi)
    kern = kc == 1 ? (BM == 128 ? thomas_tma_kernel<128, 3, 16, true> : thomas_tma_kernel<BMAX, 3, 16, true>)
           : kc == 2 ? (BM == 128 ? thomas_tma_kernel<128, 2, 16, true> : thomas_tma_kernel<BMAX, 2, 16, true>)
           : BM == 128 ? (S == 4 ? thomas_tma_kernel<128, 4, K, true> : thomas_tma_kernel<128, 3, K, true>)
                       : (S == 4 ? thomas_tma_kernel<BMAX, 4, K, true> : thomas_tma_kernel<BMAX, 3, K, true>);
  else
    kern = kc == 1 ? (BM == 128 ? thomas_tma_kernel<128, 3, 16, false> : thomas_tma_kernel<BMAX, 3, 16, false>)
           : kc == 2 ? (BM == 128 ? thomas_tma_kernel<128, 2, 16, false> : thomas_tma_kernel<BMAX, 2, 16, false>)
           : BM == 128 ? (S == 4 ? thomas_tma_kernel<128, 4, K, false> : thomas_tma_kernel<128, 3, K, false>)
                       : (S == 4 ? thomas_tma_kernel<BMAX, 4, K, false> : thomas_tma_kernel<BMAX, 3, K, false>);
  HFB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 1, sms = 148, dev = 0;
  HFB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BM, sm));
  if (max_per_sm > 0) per_sm = std::min(per_sm, max_per_sm);
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = (long long)a.nrows * a.nbpr;
  const long long blocks = std::min<long long>(work, (long long)sms * std::max(per_sm, 1));
  kern<<<(unsigned)blocks, BM, sm, st>>>(a);
  HFB_LAUNCHED();
  return HFB_OK;
}

}  // namespace hfb
