#include <algorithm>
// C-ABI entry points: plan lifetime, coefficient upload, transform / tridiag
// / full-solve drivers and status reporting. See include/helmfft_b200.h.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hfb_internal.cuh"

namespace hfb {
static thread_local cudaError_t g_last_cuda = cudaSuccess;
static std::atomic<unsigned long long> g_launches{0};
void set_last_cuda(cudaError_t e) { g_last_cuda = e; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hfb

extern "C" uint64_t hfb_launch_count(void) { return hfb::g_launches.load(); }

extern "C" void hfb_set_tuning(int key, int value) { hfb::set_tuning(key, value); }

using namespace hfb;

static int ilog2_exact(int m) {
  if (m < 2 || (m & (m - 1))) return -1;
  int k = 0;
  while ((1 << k) < m) ++k;
  return k;
}

static int build_fft_tables(int n, double2** tw, double** sn, double* scale) {
  const int M = n + 1;
  std::vector<double2> t(M);
  for (int k = 0; k < M; ++k) {
    // exp(-2 pi i k / M) with the angle reduced to [0, pi/4]-symmetric form
    const double a = 2.0 * M_PI * (double)k / (double)M;
    t[k] = make_double2(std::cos(a), -std::sin(a));
  }
  // exact values at the quarter points
  t[0] = make_double2(1.0, 0.0);
  if (M % 4 == 0) {
    t[M / 4] = make_double2(0.0, -1.0);
    t[M / 2] = make_double2(-1.0, 0.0);
    t[3 * M / 4] = make_double2(0.0, 1.0);
  } else if (M % 2 == 0) {
    t[M / 2] = make_double2(-1.0, 0.0);
  }
  std::vector<double> s(M / 2 + 1);
  for (int j = 0; j <= M / 2; ++j) s[j] = std::sin(M_PI * (double)j / (double)M);
  s[0] = 0.0;
  s[M / 2] = 1.0;
  HFB_CUDA(cudaMalloc(tw, sizeof(double2) * M));
  HFB_CUDA(cudaMalloc(sn, sizeof(double) * (M / 2 + 1)));
  HFB_CUDA(cudaMemcpy(*tw, t.data(), sizeof(double2) * M, cudaMemcpyHostToDevice));
  HFB_CUDA(cudaMemcpy(*sn, s.data(), sizeof(double) * (M / 2 + 1), cudaMemcpyHostToDevice));
  *scale = std::sqrt(2.0 / (double)M);
  return HFB_OK;
}

static int build_dense(int n, double** out) {
  const long long M = n + 1;
  std::vector<double> S((size_t)n * n);
  const double sc = std::sqrt(2.0 / (double)M);
  for (int a = 1; a <= n; ++a)
    for (int b = 1; b <= n; ++b) {
      const long long r = ((long long)a * b) % (2 * M);  // sin is 2M-periodic in r
      S[(size_t)(a - 1) * n + (b - 1)] = sc * std::sin(M_PI * (double)r / (double)M);
    }
  HFB_CUDA(cudaMalloc(out, sizeof(double) * S.size()));
  HFB_CUDA(cudaMemcpy(*out, S.data(), sizeof(double) * S.size(), cudaMemcpyHostToDevice));
  return HFB_OK;
}

namespace hfb {
// dense DST-I matrices on demand (tuning key 17 forces the dense path for
// power-of-two lengths, whose plans have none)
int ensure_dense(hfb_plan* p) {
  if (!p->dense_x) {
    int rc = build_dense(p->nx, &p->dense_x);
    if (rc) return rc;
  }
  if (!p->dense_y) return build_dense(p->ny, &p->dense_y);
  return HFB_OK;
}
}  // namespace hfb

extern "C" const char* hfb_version(void) { return "helmfft_b200 0.1.0 (sm_100a)"; }

extern "C" const char* hfb_strerror(int code) {
  switch (code) {
    case HFB_OK: return "ok";
    case HFB_ERR_ARGUMENT: return "invalid argument";
    case HFB_ERR_RANGE: return "range outside extents";
    case HFB_ERR_SINGULAR: return "vanishing pivot (singular spectral system)";
    case HFB_ERR_PARTITION: return "invalid partition";
    case HFB_ERR_EXCHANGE: return "exchange failure";
    case HFB_ERR_CUDA: return cudaGetErrorString(hfb::g_last_cuda);
    case HFB_ERR_NO_COEFFICIENTS: return "plan has no coefficients";
    default: return "unknown error";
  }
}

static void stage_events_free(hfb_plan* p) {
  for (int i = 0; i < 6 * p->stage_ring; ++i) cudaEventDestroy(p->stage_ev[i]);
  std::free(p->stage_ev);
  p->stage_ev = nullptr;
  p->stage_ring = 0;
  p->stage_count = 0;
}

extern "C" int hfb_plan_destroy(hfb_plan* p) {
  if (!p) return HFB_OK;
  cudaSetDevice(p->device);
  stage_events_free(p);
  if (p->ov_stream) {
    cudaStreamSynchronize(p->ov_stream);
    cudaStreamDestroy(p->ov_stream);
    for (int i = 0; i < 4; ++i) cudaEventDestroy(p->ov_ev[i]);
  }
  cudaFree(p->tw_x);
  cudaFree(p->sn_x);
  cudaFree(p->tw_y);
  cudaFree(p->sn_y);
  cudaFree(p->dense_x);
  cudaFree(p->dense_y);
  cudaFree(p->lvlmap);
  cudaFree(p->coef);
  cudaFree(p->coef_i);
  cudaFree(p->pq);
  cudaFree(p->ck_cache);
  cudaFree(p->cx);
  cudaFree(p->cy);
  cudaFree(p->err);
  cudaFree(p->xerr);
  cudaFree(p->ystarts);
  cudaFree(p->dev_io);
  if (p->pipe) {
    HostPipe* q = p->pipe;
    cudaStreamSynchronize(q->h2d);
    cudaStreamSynchronize(q->d2h);
    for (int b = 0; b < kPipeMax; ++b) {
      cudaFree(q->buf[b]);
      cudaEventDestroy(q->h2d_done[b]);
      cudaEventDestroy(q->solved[b]);
      cudaEventDestroy(q->d2h_done[b]);
    }
    cudaStreamDestroy(q->h2d);
    cudaStreamDestroy(q->d2h);
    delete q;
  }
  std::free(p);
  return HFB_OK;
}

extern "C" int hfb_plan_create(int nx, int ny, int nz, int device, hfb_plan** out) {
  if (!out || nx < 1 || ny < 1 || nz < 1) return HFB_ERR_ARGUMENT;
  *out = nullptr;
  hfb_plan* p = (hfb_plan*)std::calloc(1, sizeof(hfb_plan));
  if (!p) return HFB_ERR_ARGUMENT;
  p->nx = nx;
  p->ny = ny;
  p->nz = nz;
  p->device = device;
  int rc = HFB_OK;
  if (cudaSetDevice(device) != cudaSuccess) {
    std::free(p);
    return HFB_ERR_CUDA;
  }
  p->logMx = ilog2_exact(nx + 1);
  p->logMy = ilog2_exact(ny + 1);
  if (p->logMx >= 0)
    rc = build_fft_tables(nx, &p->tw_x, &p->sn_x, &p->scale_x);
  else
    rc = build_dense(nx, &p->dense_x);
  if (!rc) {
    if (p->logMy >= 0)
      rc = build_fft_tables(ny, &p->tw_y, &p->sn_y, &p->scale_y);
    else
      rc = build_dense(ny, &p->dense_y);
  }
  if (!rc && cudaMalloc(&p->err, sizeof(unsigned long long)) != cudaSuccess) rc = HFB_ERR_CUDA;
  if (!rc && cudaMemset(p->err, 0xff, sizeof(unsigned long long)) != cudaSuccess) rc = HFB_ERR_CUDA;
  if (rc) {
    hfb_plan_destroy(p);
    return rc;
  }
  *out = p;
  return HFB_OK;
}

static void scaled_table(const double* table, size_t nlev, double* buf) {
  // device layout: [scaled (4a,2b,2c,d) x nz*3][raw (a,b,c,d) x nz*3]
  for (size_t e = 0; e < nlev; e += 4) {
    buf[e + 0] = 4.0 * table[e + 0];
    buf[e + 1] = 2.0 * table[e + 1];
    buf[e + 2] = 2.0 * table[e + 2];
    buf[e + 3] = table[e + 3];
  }
  std::memcpy(buf + nlev, table, sizeof(double) * nlev);
}

extern "C" int hfb_plan_set_coefficients_z(hfb_plan* p, const double* table_re,
                                           const double* table_im, const double* cx,
                                           const double* cy, double thr) {
  if (!p || !table_im) return HFB_ERR_ARGUMENT;
  int rc = hfb_plan_set_coefficients(p, table_re, cx, cy, thr);
  if (rc) return rc;
  const size_t nlev = (size_t)p->nz * 12;
  std::vector<double> buf(2 * nlev);
  scaled_table(table_im, nlev, buf.data());
  p->zinv = 0;  // the complex z-solve keeps per-level weights
  if (!p->coef_i) HFB_CUDA(cudaMalloc(&p->coef_i, sizeof(double) * 2 * nlev));
  HFB_CUDA(cudaMemcpy(p->coef_i, buf.data(), sizeof(double) * 2 * nlev, cudaMemcpyHostToDevice));
  return HFB_OK;
}

extern "C" int hfb_plan_set_coefficients(hfb_plan* p, const double* table, const double* cx,
                                         const double* cy, double thr) {
  if (!p || !table || !cx || !cy) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  // kernels queued on any stream (torch side streams do not order against the
  // synchronous copies below) may still read the old table: let them finish
  if (p->have_coef) HFB_CUDA(cudaDeviceSynchronize());
  const size_t nlev = (size_t)p->nz * 12;
  std::vector<double> buf(2 * nlev);
  scaled_table(table, nlev, buf.data());
  if (p->coef_i) {  // a real table replaces a complex one
    cudaFree(p->coef_i);
    p->coef_i = nullptr;
  }
  if (!p->coef) HFB_CUDA(cudaMalloc(&p->coef, sizeof(double) * 2 * nlev));
  if (!p->cx) HFB_CUDA(cudaMalloc(&p->cx, sizeof(double) * p->nx));
  if (!p->cy) HFB_CUDA(cudaMalloc(&p->cy, sizeof(double) * p->ny));
  HFB_CUDA(cudaMemcpy(p->coef, buf.data(), sizeof(double) * 2 * nlev, cudaMemcpyHostToDevice));
  HFB_CUDA(cudaMemcpy(p->cx, cx, sizeof(double) * p->nx, cudaMemcpyHostToDevice));
  HFB_CUDA(cudaMemcpy(p->cy, cy, sizeof(double) * p->ny, cudaMemcpyHostToDevice));
  p->thr = thr;
  p->have_coef = 1;
  p->coef_epoch++;  // cached cp checkpoints (ck_cache) belong to the previous table
  p->ck_valid = 0;
  p->zinv = 1;  // all levels' scaled weights equal (bitwise)
  for (size_t e = 12; e < nlev && p->zinv; ++e)
    if (std::memcmp(&buf[e], &buf[e % 12], sizeof(double)) != 0) p->zinv = 0;
  return build_pq(p);
}

extern "C" int hfb_stage_timing(hfb_plan* p, int ring) {
  if (!p || ring < 0) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  stage_events_free(p);
  if (ring == 0) return HFB_OK;
  p->stage_ev = (cudaEvent_t*)std::calloc(6 * (size_t)ring, sizeof(cudaEvent_t));
  if (!p->stage_ev) return HFB_ERR_ARGUMENT;
  for (int i = 0; i < 6 * ring; ++i) {
    if (cudaEventCreate(&p->stage_ev[i]) != cudaSuccess) {
      p->stage_ring = i / 6;
      stage_events_free(p);
      return HFB_ERR_CUDA;
    }
  }
  p->stage_ring = ring;
  return HFB_OK;
}

extern "C" int hfb_stage_times(hfb_plan* p, float* ms, int* nslots) {
  if (!p || !ms || !nslots || !p->stage_ring) return HFB_ERR_ARGUMENT;
  const long long n = std::min<long long>(p->stage_count, p->stage_ring);
  for (long long r = 0; r < n; ++r) {
    cudaEvent_t* e = p->stage_ev + 6 * r;
    HFB_CUDA(cudaEventSynchronize(e[5]));
    for (int i = 0; i < 5; ++i) HFB_CUDA(cudaEventElapsedTime(&ms[5 * r + i], e[i], e[i + 1]));
  }
  *nslots = (int)n;
  return HFB_OK;
}

extern "C" int hfb_plan_set_workspace_mode(hfb_plan* p, int lean) {
  if (!p || lean < 0 || lean > 1) return HFB_ERR_ARGUMENT;
  p->ws_lean = lean;
  return HFB_OK;
}

extern "C" int hfb_plan_trim(hfb_plan* p) {
  if (!p) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  if (p->ck_cache) {
    HFB_CUDA(cudaFree(p->ck_cache));  // waits for the work that still reads it
    p->ck_cache = nullptr;
    p->ck_cache_bytes = 0;
    p->ck_valid = 0;
  }
  return HFB_OK;
}

extern "C" size_t hfb_workspace_bytes(const hfb_plan* p, int op) {
  if (!p) return 0;
  const size_t vol = (size_t)p->nx * p->ny * p->nz;
  const size_t tw = transform_work_elems(p, p->nz);
  const size_t fw = fused_work_elems(p);
  switch (op) {
    case 0: return sizeof(double) * (fw ? fw : vol + tw);  // fused, or cp + scratch
    case 1: return sizeof(double) * tw;
    case 2: return sizeof(double) * vol;
    case 3: {  // hfb_solve_z
      const size_t fz = fused_work_elems_z(p);
      return sizeof(double) * (fz ? fz : 2 * vol + tw);
    }
    case 4: return sizeof(double) * 2 * vol;  // hfb_solve_slab_z (full n_y modes)
    case 5: return sizeof(double) * modes_work_elems(p);  // hfb_forward_modes
    default: return 0;
  }
}

static int transform_range(hfb_plan* p, const double* src, double* dst, int z0, int z1,
                           double* tmp, cudaStream_t st) {
  return transform_planes(p, src, dst, z0, z1, tmp, st);
}

extern "C" int hfb_transform_stack(hfb_plan* p, double* data, int z0, int z1, void* work,
                                   void* stream) {
  const NvtxRange nvtx_("hfb_transform_stack");
  if (!p || !data) return HFB_ERR_ARGUMENT;
  if (z0 < 0 || z0 > z1 || z1 > p->nz) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return transform_range(p, data, data, z0, z1, (double*)work, (cudaStream_t)stream);
}

extern "C" int hfb_transform_lines_x(hfb_plan* p, double* data, int y0, int y1, void* work,
                                     void* stream) {
  const NvtxRange nvtx_("hfb_transform_lines_x");
  if (!p || !data) return HFB_ERR_ARGUMENT;
  if (y0 < 0 || y0 > y1 || y1 > p->ny) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_dst_x(p, data, data, 0, p->nz, y0, y1, (double*)work, (cudaStream_t)stream);
}

extern "C" int hfb_transform_lines_y(hfb_plan* p, double* data, int x0, int x1, void* work,
                                     void* stream) {
  const NvtxRange nvtx_("hfb_transform_lines_y");
  if (!p || !data) return HFB_ERR_ARGUMENT;
  if (x0 < 0 || x0 > x1 || x1 > p->nx) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_dst_y(p, data, data, 0, p->nz, x0, x1, (double*)work, (cudaStream_t)stream);
}

extern "C" int hfb_solve_slab(hfb_plan* p, double* slab, int m_count, int m_offset, void* work,
                              void* stream) {
  const NvtxRange nvtx_("hfb_solve_slab");
  if (!p || !slab || !work) return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;  // complex table: hfb_solve_slab_z
  if (m_count < 0 || m_offset < 0 || m_offset + m_count > p->ny) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas(p, slab, m_count, m_offset, (double*)work, (cudaStream_t)stream);
}

extern "C" int hfb_solve(hfb_plan* p, const double* rhs, double* out, void* work, void* stream) {
  const NvtxRange nvtx_("hfb_solve");
  if (!p || !rhs || !out || !work) return HFB_ERR_ARGUMENT;
  if (!p->have_coef) return HFB_ERR_NO_COEFFICIENTS;
  if (p->coef_i) return HFB_ERR_ARGUMENT;  // complex table: hfb_solve_z
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (fused_work_elems(p)) return solve_fused(p, rhs, out, (double*)work, st);
  const size_t vol = (size_t)p->nx * p->ny * p->nz;
  double* cpw = (double*)work;
  double* tmp = transform_work_elems(p, p->nz) ? cpw + vol : nullptr;
  const StageMarks mark(p, st);
  mark(0);
  int rc = transform_range(p, rhs, out, 0, p->nz, tmp, st);
  if (rc) return rc;
  mark(1);
  mark(2);
  rc = launch_thomas(p, out, p->ny, 0, cpw, st);
  if (rc) return rc;
  mark(3);
  mark(4);
  rc = transform_range(p, out, out, 0, p->nz, tmp, st);
  mark(5);
  return rc;
}

extern "C" int hfb_solve_slab_z(hfb_plan* p, double* re, double* im, int m_count, int m_offset,
                                void* work, void* stream) {
  const NvtxRange nvtx_("hfb_solve_slab_z");
  if (!p || !re || !im || !work) return HFB_ERR_ARGUMENT;
  if (!p->have_coef || !p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  if (m_count < 0 || m_offset < 0 || m_offset + m_count > p->ny) return HFB_ERR_RANGE;
  HFB_CUDA(cudaSetDevice(p->device));
  return launch_thomas_slab_z(p, re, im, m_count, m_offset, (double*)work, (cudaStream_t)stream);
}

extern "C" int hfb_solve_z(hfb_plan* p, const double* rhs_re, const double* rhs_im,
                           double* out_re, double* out_im, void* work, void* stream) {
  const NvtxRange nvtx_("hfb_solve_z");
  if (!p || !rhs_re || !rhs_im || !out_re || !out_im || !work) return HFB_ERR_ARGUMENT;
  if (!p->have_coef || !p->coef_i) return HFB_ERR_NO_COEFFICIENTS;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (fused_work_elems_z(p))
    return solve_fused_z(p, rhs_re, rhs_im, out_re, out_im, (double*)work, st);
  const size_t vol = (size_t)p->nx * p->ny * p->nz;
  double* cpw = (double*)work;
  double* tmp = transform_work_elems(p, p->nz) ? cpw + 2 * vol : nullptr;
  const StageMarks mark(p, st);
  mark(0);
  int rc = transform_range(p, rhs_re, out_re, 0, p->nz, tmp, st);
  if (!rc) rc = transform_range(p, rhs_im, out_im, 0, p->nz, tmp, st);
  mark(1);
  mark(2);
  if (!rc) rc = launch_thomas_slab_z(p, out_re, out_im, p->ny, 0, cpw, st);
  mark(3);
  mark(4);
  if (!rc) rc = transform_range(p, out_re, out_re, 0, p->nz, tmp, st);
  if (!rc) rc = transform_range(p, out_im, out_im, 0, p->nz, tmp, st);
  mark(5);
  return rc;
}

extern "C" int hfb_status_fetch(hfb_plan* p, void* stream, hfb_status* s) {
  if (!p) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long key = ~0ULL;
  HFB_CUDA(cudaMemcpyAsync(&key, p->err, sizeof(key), cudaMemcpyDeviceToHost, st));
  HFB_CUDA(cudaStreamSynchronize(st));
  if (s) std::memset(s, 0, sizeof(*s));
  if (key == ~0ULL) return HFB_OK;
  HFB_CUDA(cudaMemsetAsync(p->err, 0xff, sizeof(unsigned long long), st));
  HFB_CUDA(cudaStreamSynchronize(st));
  const unsigned long long nx = p->nx, ny = p->ny;
  const long long n = (long long)(key % nx);
  const long long m = (long long)((key / nx) % ny);
  const long long l = (long long)(key / (nx * ny));
  if (s) {
    s->code = HFB_ERR_SINGULAR;
    s->l = l + 1;
    s->m = m + 1;
    s->n = n + 1;
    std::snprintf(s->msg, sizeof(s->msg), "vanishing pivot at row %lld for mode (n=%lld, m=%lld)",
                  l + 1, n + 1, m + 1);
  }
  return HFB_ERR_SINGULAR;
}

extern "C" int hfb_solve_host(hfb_plan* p, const double* hin, double* hout, void* work,
                              void* stream, hfb_status* s) {
  const NvtxRange nvtx_("hfb_solve_host");
  if (!p || !hin || !hout || !work) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * (size_t)p->nx * p->ny * p->nz;
  if (p->dev_io_bytes < bytes) {
    if (p->dev_io) cudaFree(p->dev_io);
    p->dev_io = nullptr;
    p->dev_io_bytes = 0;
    HFB_CUDA(cudaMalloc(&p->dev_io, bytes));
    p->dev_io_bytes = bytes;
  }
  HFB_CUDA(cudaMemcpyAsync(p->dev_io, hin, bytes, cudaMemcpyHostToDevice, st));
  int rc = hfb_solve(p, p->dev_io, p->dev_io, work, stream);
  if (rc) return rc;
  HFB_CUDA(cudaMemcpyAsync(hout, p->dev_io, bytes, cudaMemcpyDeviceToHost, st));
  return hfb_status_fetch(p, stream, s);
}

// ---------------------------------------------------------------------------
// Pipelined host solves: H2D of call k+1 and D2H of call k-1 run on their own
// copy streams (separate copy engines) while call k solves on the caller's
// stream; two device volumes alternate. Host buffers must be pinned and stay
// valid until hfb_host_sync.
static int host_pipe(hfb_plan* p, size_t bytes) {
  if (p->pipe && p->pipe->bytes >= bytes) return HFB_OK;
  if (p->pipe) {
    HFB_CUDA(cudaStreamSynchronize(p->pipe->h2d));
    HFB_CUDA(cudaStreamSynchronize(p->pipe->d2h));
    for (int b = 0; b < kPipeMax; ++b) {
      cudaFree(p->pipe->buf[b]);
      p->pipe->buf[b] = nullptr;
    }
  } else {
    p->pipe = new HostPipe();
    HostPipe* q = p->pipe;
    HFB_CUDA(cudaStreamCreateWithFlags(&q->h2d, cudaStreamNonBlocking));
    HFB_CUDA(cudaStreamCreateWithFlags(&q->d2h, cudaStreamNonBlocking));
    for (int b = 0; b < kPipeMax; ++b) {
      HFB_CUDA(cudaEventCreateWithFlags(&q->h2d_done[b], cudaEventDisableTiming));
      HFB_CUDA(cudaEventCreateWithFlags(&q->solved[b], cudaEventDisableTiming));
      HFB_CUDA(cudaEventCreateWithFlags(&q->d2h_done[b], cudaEventDisableTiming));
      HFB_CUDA(cudaEventRecord(q->d2h_done[b], q->d2h));
    }
  }
  HostPipe* q = p->pipe;
  q->bytes = 0;
  q->next = 0;
  for (int b = 0; b < 2; ++b) HFB_CUDA(cudaMalloc(&q->buf[b], bytes));
  q->nbuf = 2;
  // a third volume only with room to spare (the solve's workspace is already
  // allocated by the caller)
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b > bytes + (bytes >> 3) &&
      cudaMalloc(&q->buf[2], bytes) == cudaSuccess)
    q->nbuf = 3;
  cudaGetLastError();  // a refused third volume is not an error
  q->bytes = bytes;
  return HFB_OK;
}

extern "C" int hfb_solve_host_async(hfb_plan* p, const double* hin, double* hout, void* work,
                                    void* stream) {
  const NvtxRange nvtx_("hfb_solve_host_async");
  if (!p || !hin || !hout || !work) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * (size_t)p->nx * p->ny * p->nz;
  int rc = host_pipe(p, bytes);
  if (rc) return rc;
  HostPipe* q = p->pipe;
  const int b = q->next;
  q->next = (b + 1) % q->nbuf;
  HFB_CUDA(cudaStreamWaitEvent(q->h2d, q->d2h_done[b], 0));
  HFB_CUDA(cudaMemcpyAsync(q->buf[b], hin, bytes, cudaMemcpyHostToDevice, q->h2d));
  HFB_CUDA(cudaEventRecord(q->h2d_done[b], q->h2d));
  HFB_CUDA(cudaStreamWaitEvent(st, q->h2d_done[b], 0));
  if ((rc = hfb_solve(p, q->buf[b], q->buf[b], work, stream))) return rc;
  HFB_CUDA(cudaEventRecord(q->solved[b], st));
  HFB_CUDA(cudaStreamWaitEvent(q->d2h, q->solved[b], 0));
  HFB_CUDA(cudaMemcpyAsync(hout, q->buf[b], bytes, cudaMemcpyDeviceToHost, q->d2h));
  HFB_CUDA(cudaEventRecord(q->d2h_done[b], q->d2h));
  return HFB_OK;
}

extern "C" int hfb_host_sync(hfb_plan* p, hfb_status* s) {
  if (!p) return HFB_ERR_ARGUMENT;
  HFB_CUDA(cudaSetDevice(p->device));
  if (!p->pipe) return hfb_status_fetch(p, nullptr, s);
  HFB_CUDA(cudaStreamSynchronize(p->pipe->h2d));
  HFB_CUDA(cudaStreamSynchronize(p->pipe->d2h));
  return hfb_status_fetch(p, p->pipe->d2h, s);
}
