/*
 * helmfft_b200.h — C-ABI of the B200 (sm_100a) hot path of the arXiv 1912.03565
 * direct solver: forward orthonormal 2D DST-I of every z-plane, N_x*N_y
 * independent tridiagonal (Thomas) solves along z, inverse 2D DST-I, plus the
 * compact-scheme RHS operators and the 27-point operator used for folding and
 * residuals.
 *
 * The reference (`helmfft`, pure Python on numpy/scipy) has no FFI; its
 * boundary is the Python API. Each entry point below replaces one reference
 * operator and is bound from Python through ctypes
 * (paper_1912_03565_b200/_native.py; INTEGRATION.md shows the stub a helmfft
 * maintainer would add). Conventions:
 *
 *  - every array is fp64 real, C order (n_z, n_y, n_x), x fastest — the
 *    row ordering of reference assembly.py:32-34 / oracle.py:27-29;
 *  - device pointers are borrowed for the duration of the call; all work is
 *    enqueued on `stream` (a cudaStream_t passed as void*, NULL = legacy);
 *  - workspaces are allocated by the caller (PyTorch) with the size that
 *    hfb_workspace_bytes() reports;
 *  - calls return an hfb_code; singular pivots are detected on the device and
 *    reported by hfb_status_fetch() (the only synchronising call).
 */
#ifndef HELMFFT_B200_H
#define HELMFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HFB_OK = 0,
  HFB_ERR_ARGUMENT = 1,      /* ValueError: shapes, extents            */
  HFB_ERR_RANGE = 2,         /* IndexError: plane / pencil ranges      */
  HFB_ERR_SINGULAR = 3,      /* SingularSystemError(n, m)              */
  HFB_ERR_PARTITION = 4,     /* InvalidPartitionError                  */
  HFB_ERR_EXCHANGE = 5,      /* ExchangeError(sender, receiver)        */
  HFB_ERR_CUDA = 6,          /* CUDA runtime failure                   */
  HFB_ERR_NO_COEFFICIENTS = 7
} hfb_code;

/* Error payload; mirrors the reference exceptions (errors.py:1-31). */
typedef struct {
  int code;
  int64_t l;        /* 1-based row level of the vanishing pivot            */
  int64_t m;        /* 1-based global sine mode along y                   */
  int64_t n;        /* 1-based sine mode along x                          */
  int sender;
  int receiver;
  char msg[256];
} hfb_status;

typedef struct hfb_plan hfb_plan;

/* Library version string. */
const char* hfb_version(void);

/* Human-readable text for an hfb_code. */
const char* hfb_strerror(int code);

/* Number of kernels this library has launched in the process (all plans). */
uint64_t hfb_launch_count(void);

/* Performance knobs (no effect on results beyond rounding: keys 0, 17 and 18
 * change the transform's factorisation; every other knob keeps the bits, except
 * key 20's reordered residual sum). They are process-wide (every plan,
 * every thread) and read when a kernel is launched: set them before the solves
 * they should affect, not concurrently with them. key 0 = DST engine width
 * (16 or 32 values per thread), key 1 = transform groups per CTA (0 = auto),
 * key 2 = L2 promotion of the column (tensor-box) loads: 0 none, 1 64 B,
 * 2 128 B (default), 3 256 B; key 3 = batch order: 0 auto (interleaved over
 * CTAs; column passes in runs of one 128-byte line), 1 one contiguous run per
 * CTA, R >= 2 interleaved runs of R batches; key 4 = row outputs by TMA
 * tensor stores where the destination layout allows (1, default) or by
 * thread stores (0); key 5 = fuse the forward Thomas sweep into the one-call
 * solve's y-pass (1) or not (0, default: the carried per-mode state limits the
 * fused kernel to 8 warps per SM, 12 ms against 4 + 3 ms unfused); key 6 =
 * overlap the z-solve with the y-passes on a second stream, halves of the
 * x-modes (1) or not (0, default: the CTA caps that make room for both cost
 * more than the overlap gains, 22.5 vs 21.7 ms at 1023^3), keys 7 / 8 = those
 * caps (CTAs per SM of the y-passes / of the z-solve); key 9 = write packed
 * rows (the user's array) by row-pair 1D bulk stores (1) or thread stores (0,
 * default: the register rotation it needs costs more than it saves); key 10 =
 * cap on resident CTAs per SM for every DST pass (0, default: occupancy);
 * key 11 = how long the distributed z-solve waits for a neighbour's carry
 * before latching an exchange error, in ms (0, default: 30000); key 12 = CTAs
 * per SM of the distributed z-solve (0, default: occupancy; 1 or 2 deepen its
 * copy ring); key 13 = write packed rows (the user's odd-pitch array) by 2D
 * tensor stores of the destination viewed as flat 128-byte rows, head and tail
 * by plain stores (1, default) or by thread stores (0); key 14 = row passes
 * with tensor stores run the transform groups of a CTA decoupled (own prefetch,
 * mbarrier and store; 1, default) or in CTA lockstep (0); key 16 = dense DST-I
 * products (lengths without an FFT) on the FP64 tensor cores (1, default) or
 * CUDA cores (0); key 17 = force the dense product for lines up to this length
 * (0, default: never; a measurement knob); key 18 = whole-plane 2D DST-I on the
 * FP64 tensor cores for lines up to this length (32, default; lines of 16 and
 * more where the FFT engine applies; 0 = never); key 19 = one-call z-solve with
 * whole columns in shared memory when n_z <= 256 and the modes fit in four
 * waves (1, default) or always the TMA copy ring (0); key 20 = levels per CTA of
 * the marching stencil kernels: the 4th-order RHS operator, the 27-point apply
 * and the residual (32, default; 0 = the per-point gather kernels); key 21 = the
 * one-call solve's wavefront-fused z-solve (forward elimination inside the
 * y-pass, back substitution inside the inverse y-pass, carries through L2 with
 * per-block level counters; fast layout, y-lines of 511 / 1023; bitwise equal;
 * 0, default: measured slower); key 22 = its measurement variants;
 * key 23 = the TMA z-solve stores x' only at the first level of each 8-level
 * chunk and recomputes the rest in the back substitution (1, default: 27
 * instead of 34 B/point) or every level (0); key 24 = levels per CTA of the
 * plane-streamed 27-point apply / fold / residual (32, default; 0 = key 20's
 * kernels); key 25 = their rows per warp without shared memory (2 or 4,
 * default 4); key 26 = ring stages of the TMA z-solve (3, default, or 4);
 * key 27 = the streamed 27-point kernels stage their planes in shared memory
 * by cp.async (1, default) or read them from registers (0); key 28 = TMA
 * z-solve blocks of 128 modes everywhere (1) or 256 where the slab is wide
 * (0, default); key 29 = the DST passes prefetch the next batch after the
 * current one's pre-processing: 1 every pass, 2 (default) the M = 1024 passes
 * that store into the user's odd-pitch array, 0 none; key 30 = TMA z-solve chunks
 * of 16 levels with 3 (1) or 2 (2) stages, or 8 levels (0, default); key 31 =
 * z-invariant weight tables (every level's weights bitwise equal) get their
 * eigenvalues once per mode block in the z-solves (1, default) or per level
 * (0); key 32 = the one-call z-solve keeps its cp checkpoints (matrix-only data,
 * one plane per 8 levels) in a plan-owned array across solves with the same
 * coefficients, so only the first solve after a coefficient upload writes them
 * (1, default; 0 = every solve writes them into the caller's workspace).
 * Key 14 = 2 also decouples the groups of the flat-row-store column pass.
 * Keys 5, 6, 9, 21, 26 = 4, 28 and 30 keep measured-slower variants for A/B
 * runs; keys 17 and 22 are measurement knobs (22 bit 0 skips the waits: wrong
 * results). All of them keep the bits of the default path except keys 0, 17,
 * 18 and the residual order of 20 / 24 / 27. */
void hfb_set_tuning(int key, int value);

/* Plan for an (n_z, n_y, n_x) interior grid on CUDA device `device`.
 * Replaces spectral.make_plan (spectral.py:46-51) and carries the per-row
 * coefficient table that tridiag.solve_slab builds on every call
 * (tridiag.py:112-123). Twiddle, sine and (for N+1 not a power of two)
 * dense DST-I tables are built here. */
int hfb_plan_create(int n_x, int n_y, int n_z, int device, hfb_plan** out);
int hfb_plan_destroy(hfb_plan* plan);

/* Upload the row coefficient table and mode cosines.
 * table: n_z * 12 doubles, row l (0-based) holds, for level offset k = 0,1,2
 *        (levels l-1, l, l+1), the weights (a, b, c, d) — i.e.
 *        table[l*12 + k*4 + {0,1,2,3}] = A[l,k], B[l,k], C[l,k], D[l,k]
 *        of stencil.coefficient_table (stencil.py:177-195);
 * cx: n_x cosines cos(pi n/(n_x+1)), cy: n_y cosines (stencil.py:219-223);
 * pivot_threshold: PIVOT_RTOL * max|table| (tridiag.py:22, 136-137). */
int hfb_plan_set_coefficients(hfb_plan* plan, const double* table, const double* cx,
                              const double* cy, double pivot_threshold);

/* Workspace sizes in bytes. op: 0 = hfb_solve, 1 = hfb_transform_stack,
 * 2 = hfb_solve_slab (for the full n_y modes), 3 = hfb_solve_z,
 * 4 = hfb_solve_slab_z (full n_y), 5 = hfb_forward_modes. */
size_t hfb_workspace_bytes(const hfb_plan* plan, int op);

/* Layout of the hfb_solve workspace (no effect on results): 0 = fast (two
 * padded scratch volumes; every DST pass reads and writes whole rows or
 * tensor-map column boxes), 1 = lean (one padded scratch volume; the forward
 * x-pass writes transposed). hfb_workspace_bytes(plan, 0) reports the size for
 * the current mode, which hfb_solve then expects. Default 0. */
int hfb_plan_set_workspace_mode(hfb_plan* plan, int lean);

/* Give back the device memory the plan allocated on its own for reuse across
 * solves: the z-solve's cached cp checkpoints (tuning key 32; one plane per 8
 * levels, 1.07 GB at 1023^3). The next hfb_solve allocates and fills them again.
 * For callers that keep many plans alive and run short of memory. */
int hfb_plan_trim(hfb_plan* plan);

/* Per-stage CUDA events of the one-call solve (measurement only). With a ring
 * of R > 0 slots, each hfb_solve records an event before its first and after
 * each of its five launches on the caller's stream, in slot (solve count mod
 * R); R = 0 disables and frees them. hfb_stage_times waits for the recorded
 * slots and writes 5 durations (ms) per slot — the x-pass, y-pass, z-solve,
 * inverse y-pass and inverse x-pass of DESIGN.md §4 — and the number of
 * recorded slots (ms must hold 5 R floats). */
int hfb_stage_timing(hfb_plan* plan, int ring);
int hfb_stage_times(hfb_plan* plan, float* ms, int* nslots);

/* Orthonormal 2D DST-I (x-pass then y-pass) of planes [z0, z1) in place.
 * Replaces spectral.transform_stack (spectral.py:75-91). */
int hfb_transform_stack(hfb_plan* plan, double* data, int z0, int z1, void* work,
                        void* stream);

/* 1D passes on all planes, restricted to a y-range (x-pass) or an x-range
 * (y-pass). Replace spectral.transform_lines_x/y (spectral.py:94-111). */
int hfb_transform_lines_x(hfb_plan* plan, double* data, int y0, int y1, void* work,
                          void* stream);
int hfb_transform_lines_y(hfb_plan* plan, double* data, int x0, int x1, void* work,
                          void* stream);

/* Thomas sweep over a (n_z, m_count, n_x) slab in place; local row j is
 * global mode m_offset + j. Replaces tridiag.solve_slab/_sweep
 * (tridiag.py:112-167). Pivot failures are latched for hfb_status_fetch. */
int hfb_solve_slab(hfb_plan* plan, double* slab, int m_count, int m_offset, void* work,
                   void* stream);

/* Batched Thomas on explicit bands (tridiag.solve_system, tridiag.py:59-90):
 * sub/diag/sup/x are (nsys, n) doubles, or (nsys, n) interleaved complex when
 * is_complex != 0; x is overwritten with the solution; cp_ws has x's size.
 * thr[s] = PIVOT_RTOL * max band magnitude of system s; the first vanishing
 * pivot is latched into *err as s*n + row (caller initialises *err = ~0). */
int hfb_solve_bands(const double* sub, const double* diag, const double* sup, double* x,
                    double* cp_ws, int n, int nsys, int is_complex, const double* thr,
                    unsigned long long* err, void* stream);

/* Full solve: U = V_z-solve(V F), V = 2D DST-I. rhs and out may alias
 * (in place). Replaces the Sequential/SharedWorkers branch of
 * solver.solve_discrete (solver.py:293-317) after the Dirichlet fold. */
int hfb_solve(hfb_plan* plan, const double* rhs, double* out, void* work, void* stream);

/* Same as hfb_solve with host (ideally pinned) buffers: H2D, solve, D2H,
 * synchronised, pivot status reported in *status (may be NULL). */
int hfb_solve_host(hfb_plan* plan, const double* host_rhs, double* host_out, void* work,
                   void* stream, hfb_status* status);

/* Synchronise `stream`, report (and clear) a latched singular pivot. */
int hfb_status_fetch(hfb_plan* plan, void* stream, hfb_status* status);

/* Pipelined host-buffer solves for many right-hand sides (serving / time
 * stepping): each call enqueues H2D of host_rhs, the solve (on `stream`) and
 * D2H into host_out, and returns without waiting. The H2D of the next call and
 * the D2H of the previous one run on the plan's own copy streams while this
 * one solves; three device volumes rotate (two when a third does not fit),
 * so a call's H2D never waits for the previous call's D2H. Host buffers must be pinned and
 * stay untouched until hfb_host_sync, which waits for every pending call and
 * reports a latched pivot failure like hfb_status_fetch. */
int hfb_solve_host_async(hfb_plan* plan, const double* host_rhs, double* host_out, void* work,
                         void* stream);
int hfb_host_sync(hfb_plan* plan, hfb_status* status);

/* Fourth-order RHS operator F = h_z^2 (f/2 + (1/12) sum of the 6 face
 * neighbours) of f sampled on the closed (n_z+2, n_y+2, n_x+2) grid.
 * Replaces the FOURTH_ORDER branch of assembly.build_rhs (assembly.py:183-193). */
int hfb_rhs_fourth(hfb_plan* plan, const double* f_closed, double* rhs, double h_z2,
                   void* stream);

/* Pointwise RHS combinations of sampled fields (assembly.py:180-181, 195-224).
 * kind 2: F = hz2*f. kind 6: fields = {f, lap_f, d4_f, f_xxyy, f_xxzz, f_yyzz,
 * f_z}, params = {h2, k2[1..nz] ptr unused}. See hfb_rhs_sixth/cd4. */
int hfb_rhs_second(hfb_plan* plan, const double* f, double* rhs, double h_z2, void* stream);
int hfb_rhs_sixth(hfb_plan* plan, const double* f, const double* lap, const double* d4,
                  const double* fxxyy, const double* fxxzz, const double* fyyzz,
                  const double* fz, const double* k2_levels /* n_z */,
                  const double* k2z_levels /* n_z */, double h2, double* rhs, void* stream);
int hfb_rhs_convdiff(hfb_plan* plan, const double* f, const double* fxx, const double* fyy,
                     const double* fz, const double* fzz, double hx2, double hy2, double hz2,
                     double gamma, double* rhs, void* stream);

/* 27-point operator on a closed-box array ext (n_z+2, n_y+2, n_x+2):
 * out = A*ext restricted to the interior, with the reference's term order and
 * zero-column skipping (assembly.py:229-244). term_mask bit (k*9 + o) enables
 * level offset k (0..2) and plane offset o in the order a(-1,-1),(1,-1),(-1,1),
 * (1,1), b(-1,0),(1,0), c(0,-1),(0,1), d(0,0). mode 0: out = A ext;
 * mode 1: out = rhs - A ext (Dirichlet fold, assembly.py:258-274). */
int hfb_apply27(hfb_plan* plan, const double* ext, const double* rhs, double* out,
                uint32_t term_mask, int mode, void* stream);

/* Sum of squares of (A*u - F) with zero boundary (assembly.py:277-289):
 * u, F interior arrays; partial sums written to `partial` (length returned by
 * hfb_residual_partials()). */
int hfb_residual_partials(const hfb_plan* plan);
int hfb_residual_sq(hfb_plan* plan, const double* u, const double* rhs, double* partial,
                    uint32_t term_mask, void* stream);

/* ---- complex k(z): complex weight tables -------------
 * The reference computes in complex128 throughout (grid.py:8-9, 126-129);
 * complex fields travel as two real volumes (real, imaginary parts) in the
 * usual C-order (n_z, n_y, n_x) layout.
 *
 * Complex row table: table_re / table_im hold the real and imaginary parts in
 * the layout of hfb_plan_set_coefficients (stencil.coefficient_table with
 * complex k^2, stencil.py:177-195); pivot_threshold = PIVOT_RTOL * max|entry|.
 * A plan with a complex table rejects the real hfb_solve / hfb_solve_slab
 * (HFB_ERR_ARGUMENT); hfb_plan_set_coefficients makes it real again. */
int hfb_plan_set_coefficients_z(hfb_plan* plan, const double* table_re, const double* table_im,
                                const double* cx, const double* cy, double pivot_threshold);

/* One-call complex solve (solver.solve_discrete with complex k, solver.py:
 * 278-317): forward 2D DST of both parts, complex per-mode Thomas along z
 * (tridiag.py:126-167 in complex arithmetic), inverse 2D DST. Workspace:
 * hfb_workspace_bytes(plan, 3). Pivot failures are latched for
 * hfb_status_fetch. */
int hfb_solve_z(hfb_plan* plan, const double* rhs_re, const double* rhs_im, double* out_re,
                double* out_im, void* work, void* stream);

/* Complex per-mode solves on a transformed natural-layout y-slab (solve_slab,
 * tridiag.py:112-167). Workspace: 2 * m_count * n_x * n_z doubles
 * (hfb_workspace_bytes(plan, 4) for the full n_y). */
int hfb_solve_slab_z(hfb_plan* plan, double* re, double* im, int m_count, int m_offset,
                     void* work, void* stream);

/* Complex right-hand sides (assembly.build_rhs with complex k^2 or complex
 * gamma, assembly.py:195-224): fields_re / fields_im are arrays of the real and
 * imaginary parts of the sampled fields, in the order of hfb_rhs_sixth
 * (f, lap_f, d4_f, f_xxyy, f_xxzz, f_yyzz, f_z) or hfb_rhs_convdiff
 * (f, f_xx, f_yy, f_z, f_zz); k2 / k2z are the interior-level profiles. */
int hfb_rhs_sixth_z(hfb_plan* plan, const double* const* fields_re,
                    const double* const* fields_im, const double* k2_re, const double* k2_im,
                    const double* k2z_re, const double* k2z_im, double h2, double* F_re,
                    double* F_im, void* stream);
int hfb_rhs_convdiff_z(hfb_plan* plan, const double* const* fields_re,
                       const double* const* fields_im, double hx2, double hy2, double hz2,
                       double gamma_re, double gamma_im, double* F_re, double* F_im,
                       void* stream);

/* hfb_apply27 / hfb_residual_sq with the complex table: complex fields as
 * (re, im) pairs, each term w*v added in the reference's order. */
int hfb_apply27_z(hfb_plan* plan, const double* ext_re, const double* ext_im,
                  const double* rhs_re, const double* rhs_im, double* out_re, double* out_im,
                  uint32_t term_mask, int mode, void* stream);
int hfb_residual_sq_z(hfb_plan* plan, const double* u_re, const double* u_im,
                      const double* rhs_re, const double* rhs_im, double* partial,
                      uint32_t term_mask, void* stream);

/* z-slab -> send-buffer pack and receive-buffer -> z-slab unpack for the
 * partitioned exchange (solver.py:146-201). y_starts has parts+1 entries
 * (prefix of the y-ranges). Forward: send[q] = slab[:, y-range(q), :]
 * contiguous, blocks concatenated in ascending q. Inverse: recv blocks
 * (kpz, kpy(q), n_x) concatenated in ascending q -> slab[:, y-range(q), :]. */
int hfb_pack_yblocks(hfb_plan* plan, const double* slab, double* send, int kpz,
                     const int* y_starts, int parts, void* stream);
int hfb_unpack_yblocks(hfb_plan* plan, const double* recv, double* slab, int kpz,
                       const int* y_starts, int parts, void* stream);

/* ---- mode-space partitioned solve (solver.py:319-399) ----
 * One rank's transformed z-slab lives as padded mode rows (kpz, n_x, ldm),
 * ldm = hfb_modes_ld(plan) (even), element (l, n, m) at (l*n_x + n)*ldm + m.
 * The exchange block for rank q is (kpz, n_x, kp(q)), kp(q) = the y-mode
 * count of q rounded up to even, blocks concatenated in ascending q; the
 * receiver's concatenation over senders is its y-slab of mode rows
 * (n_z, n_x, kp), which hfb_solve_modes streams directly.
 *   hfb_forward_modes: forward 2D DST, natural (kpz, n_y, n_x) -> mode rows
 *     (workspace hfb_workspace_bytes(plan, 5));
 *   hfb_inverse_modes: mode rows (overwritten) -> natural out;
 *   hfb_solve_modes: z-solve of a y-slab of mode rows (n_z levels of the plan,
 *     row stride ld even, columns = y-modes m_offset .. m_offset + m_count - 1),
 *     cp_work = ceil(n_z / 8) * n_x * ld doubles;
 *   hfb_pack_modes / hfb_unpack_modes: mode rows <-> exchange blocks;
 *   hfb_forward_blocks / hfb_inverse_blocks: the transforms with the exchange
 *     layout on their far side, so no pack / unpack pass runs — the forward y-pass
 *     stores every mode row straight into the blocks of `send` (one 5D tensor
 *     store per line pair), the inverse y-pass gathers its rows from the blocks of
 *     `back` (one bulk copy per block and row) into `modes` (scratch of
 *     kpz * n_x * ldm doubles). Same bits as forward_modes + pack_modes /
 *     unpack_modes + inverse_modes. They need the uniform exchange geometry —
 *     y_starts[q] = q * kp with parts * kp = n_y + 1 and kp a multiple of 16
 *     (every power-of-two n_y + 1 split over a power-of-two rank count) — and
 *     return HFB_ERR_PARTITION otherwise (callers then use the pack path). This
 *     replaces the strided block copies of exchange_forward / exchange_inverse
 *     (reference solver.py:146-201). */
int hfb_modes_ld(const hfb_plan* plan);
int hfb_forward_modes(hfb_plan* plan, const double* src, double* modes, void* work, void* stream);
int hfb_inverse_modes(hfb_plan* plan, double* modes, double* out, void* stream);
int hfb_solve_modes(hfb_plan* plan, double* data, int ld, int m_count, int m_offset,
                    void* cp_work, void* stream);
/* hfb_solve_modes on a y-slab whose levels are stored out of order (the
 * chunked exchange lands them chunk by chunk): level l lives at plane
 * level_plane[l] (host array of n_z ints, copied on `stream`). */
int hfb_solve_modes_perm(hfb_plan* plan, double* data, int ld, int m_count, int m_offset,
                         const int* level_plane, void* cp_work, void* stream);
int hfb_pack_modes(hfb_plan* plan, const double* modes, double* send, const int* y_starts,
                   int parts, void* stream);
int hfb_unpack_modes(hfb_plan* plan, const double* recv, double* modes, const int* y_starts,
                     int parts, void* stream);
int hfb_forward_blocks(hfb_plan* plan, const double* src, double* send, void* work,
                       const int* y_starts, int parts, void* stream);
int hfb_inverse_blocks(hfb_plan* plan, const double* back, double* modes, double* out,
                       const int* y_starts, int parts, void* stream);

/* ---- transpose-free distributed z-solve ("alternative to
 * measure next"; replaces the exchange_forward / solve / exchange_inverse
 * sequence of the reference's Partitioned branch, solver.py:319-399) ----
 * Every rank keeps its z-slab of mode rows (levels [z0, z0 + nzl) of the
 * plan's n_z, layout of hfb_forward_modes, row stride ld = hfb_modes_ld) and
 * the per-mode tridiagonal systems are swept across the ranks: the forward
 * elimination (dir 0) takes (x', cp) at level z0 - 1 from rank p - 1 and
 * hands its own last level to rank p + 1; the back substitution (dir 1) takes
 * W at level z0 + nzl from rank p + 1 and hands W at z0 to rank p - 1. The
 * carries move per 256-mode block through peer memory: the kernel stores into
 * the neighbour's carry region and publishes each block by a release store of
 * `epoch` into the neighbour's flag; the receiving CTA spins on it. One
 * `epoch` per solve, the same on every rank, increasing (flags start at 0).
 *   hfb_carry_layout: doubles of one rank's carry region (zero it once) and the
 *     number of flag blocks;
 *   hfb_zsolve_carry: `mine` = this rank's region, `peer` = the next rank's
 *     (dir 0) or the previous rank's (dir 1), NULL exactly when there is none;
 *     cp_work = ceil(nzl / 8) * n_x * ld doubles, shared by both directions;
 *     the plan is the full-grid plan (coefficients of all n_z levels);
 *   hfb_carry_check: synchronises `stream`; HFB_ERR_EXCHANGE when a carry never
 *     arrived within the timeout (tuning key 11, ms; default 30 s), *code = 1
 *     (forward carry from rank p - 1) or 2 (backward carry from rank p + 1);
 *   hfb_ipc_handle / hfb_ipc_open / hfb_ipc_close: CUDA IPC of a device pointer
 *     inside a larger allocation (64-byte handle + offset), for mapping the
 *     neighbours' regions in a one-process-per-GPU run. */
int hfb_carry_layout(hfb_plan* plan, int ld, long long* region_doubles, int* blocks);
int hfb_zsolve_carry(hfb_plan* plan, int dir, double* modes, int ld, int z0, int nzl,
                     void* cp_work, double* mine, double* peer, uint32_t epoch, void* stream);
/* Verification of the cross-rank carry protocol on ONE device (no peer GPUs):
 * the direction-`dir` sweeps of `nranks` virtual ranks run in ONE cooperative
 * launch, so every rank's CTAs spin on flags that the neighbouring rank's CTAs
 * publish while running concurrently (the live release/acquire path of
 * hfb_zsolve_carry across GPUs). Rank r owns levels [z0s[r], z0s[r] + nzls[r])
 * (consecutive, covering the plan's n_z), its mode rows modes[r], checkpoints
 * cp_works[r] and carry region regions[r] (hfb_carry_layout, zeroed); the peer
 * of rank r is regions[r + 1] (dir 0) or regions[r - 1] (dir 1). Synchronises
 * `stream`. Replaces nothing in the reference: it stands in for the P-GPU run
 * of solver.py:319-399 where only one GPU is available. */
int hfb_zsolve_carry_vranks(hfb_plan* plan, int dir, int nranks, double* const* modes, int ld,
                            const int* z0s, const int* nzls, void* const* cp_works,
                            double* const* regions, uint32_t epoch, void* stream);
/* The same for a complex table (complex k(z), hfb_plan_set_coefficients_z): the
 * slab travels as real and imaginary mode-row volumes (each from
 * hfb_forward_modes), cp_work = 2 * ceil(nzl / 8) * n_x * ld doubles, and the
 * carry region holds complex carries (hfb_carry_layout_z). Same arithmetic as
 * hfb_solve_z's z-solve, bit for bit. */
int hfb_carry_layout_z(hfb_plan* plan, int ld, long long* region_doubles, int* blocks);
int hfb_zsolve_carry_z(hfb_plan* plan, int dir, double* modes_re, double* modes_im, int ld,
                       int z0, int nzl, void* cp_work, double* mine, double* peer,
                       uint32_t epoch, void* stream);
int hfb_carry_check(hfb_plan* plan, void* stream, int* code);
int hfb_ipc_handle(const void* ptr, void* handle, long long* offset);
int hfb_ipc_open(const void* handle, long long offset, void** ptr);
int hfb_ipc_close(void* ptr, long long offset);

#ifdef __cplusplus
}
#endif
#endif /* HELMFFT_B200_H */
