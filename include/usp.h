/*
 * usp.h -- C-ABI of libusp: the B200 hot path of the universal split
 * preconditioner (Vettenburg & Vellekoop, arXiv 2207.14222; PAPER.md =
 * /root/reference/PAPER.md, cited by line).
 *
 * The library runs the preconditioned fixed-point (Richardson) iteration of
 * Algorithm 1 with the forward operator eliminated (Eq. 5,
 * L73-77):
 *
 *     Delta_k = B [ (L+1)^-1 (B x_k + s) - x_k ],   x_{k+1} = x_k + alpha Delta_k,
 *     stop when ||Delta_k|| / ||B (L+1)^-1 s|| < tol          (L87, reading R-4)
 *
 * with B = 1 - V (L73), (L+1)^-1 applied as a Fourier multiplier (Eq. 12,
 * L168-172) by hand-written sm_100a FFT kernels (no cuFFT), in complex64.
 * The plan runs this literal form while r_k >= r_switch and then the
 * mathematically identical Delta-recurrence of L613 (readings R-17,
 * R-30), which keeps fp32 accurate near convergence:
 *     Delta_{k+1} = Delta_k + alpha B[(L+1)^-1(B Delta_k) - Delta_k].
 *
 * Problem form (reading R-1, §2.2):
 *     A_raw = -D lap + w(r),   L_raw = -D lap + sigma,   V_raw = w - sigma,
 *     A = A_raw / c,  L = L_raw / c,  V = V_raw / c,  s = S / c,
 *     (L+1)^-1 = F^-1 [ c / (D |p|^2 + sigma + c) ] F,   p = 2 pi fftfreq(n, h).
 * Helmholtz (Eq. 8, lap psi + k^2 psi = -S): the medium is
 * k^2(r) and w = -k^2, sigma = -kbar^2, D = 1, c = -i r / target_norm (the
 * paper's c = i r/0.95 for the equation multiplied by -1).  Steady diffusion
 * (§3.2, scalar D, -D lap u + mu_a u = S): the medium is w = mu_a,
 * sigma = mu0, c = r / target_norm.
 *
 * Layout: every field is C-ordered [z][y][x], x fastest; n[0] = nx, n[1] = ny,
 * n[2] = nz (unused extents = 1).  Complex values are interleaved
 * (re, im) float32 pairs ("complex64").  Extents must be powers of two in
 * [16, 2048] (1-D: [16, 2048]; a 1-D grid is one line, solved by one CTA).
 *
 * Ownership: input pointers are borrowed for the duration of the call only
 * (their contents are copied into the workspace or consumed).  The workspace
 * is caller-owned device memory (e.g. a torch uint8 tensor), >= the size
 * usp_plan_workspace_size reports, 256-byte aligned, and must outlive the
 * plan.  The plan itself only allocates small tables and state (< 1 MiB).
 * All device work is enqueued on desc.stream.  Calls are not thread-safe per
 * plan; distinct plans are independent.
 *
 * Errors: every call returns a usp_status; nothing aborts, exits or throws
 * across the ABI.  On error usp_last_error() returns a thread-local message.
 */
#ifndef USP_H
#define USP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define USP_VERSION_MAJOR 0
#define USP_VERSION_MINOR 3

typedef struct usp_plan_s *usp_plan_t;

typedef enum {
    USP_OK = 0,
    USP_ERR_ARG = 1,             /* bad argument (NULL, size, alignment, tol...)      */
    USP_ERR_STATE = 2,           /* call out of order (e.g. iterate before source)    */
    USP_ERR_NOT_CONTRACTIVE = 3, /* max |V| >= 1: Theorem 1 needs ||V|| < 1 (L58)      */
    USP_ERR_NOT_ACCRETIVE = 4,   /* Re(w/c) < 0 somewhere or D Re(c) < 0 (Eq. 1)  */
    USP_ERR_UNSUPPORTED = 5,     /* extent not a power of two in [16,2048], ...        */
    USP_ERR_NOMEM = 6,           /* workspace too small / allocation failed            */
    USP_ERR_CUDA = 7,            /* a CUDA runtime call failed                         */
    USP_ERR_NCCL = 8,            /* an NCCL call failed                                */
    USP_ERR_NONFINITE = 9        /* non-finite values in the medium or source          */
} usp_status;

typedef enum {
    USP_CONVERGED = 0, /* r_k < tol: Algorithm 1's "until" fired (L87)                  */
    USP_MAX_ITER = 1,  /* n_max iterations ran (always the outcome when tol <= 0)       */
    USP_DIVERGED = 2   /* r_k non-finite or > 1e6 (cannot happen for valid input, Cor.1) */
} usp_term;

typedef enum {
    USP_MEDIUM_K2 = 0, /* medium array holds k^2(r) (Helmholtz); w = -k^2               */
    USP_MEDIUM_W = 1   /* medium array holds w(r) directly (diffusion: mu_a)              */
} usp_medium;

typedef enum {
    USP_C64 = 0, /* medium / source / field arrays are complex64 (interleaved float32)    */
    USP_R32 = 1  /* real float32 arrays (imaginary part 0); the field returned is real    */
} usp_dtype;

typedef enum { USP_DEVICE = 0, USP_HOST = 1, USP_STAGED = 2 /* see usp_stage_inputs */ } usp_where;

typedef struct { double re, im; } usp_c128;

typedef struct {
    int ndim;            /* 1, 2 or 3                                                     */
    int64_t n[3];        /* extents, n[0] = x (fastest)                                   */
    double h[3];         /* grid spacing per axis (p_a = 2 pi m / (n_a h_a))               */
    usp_medium medium;   /* how set_potential interprets its array                        */
    usp_dtype dtype;     /* element type of medium, source and field arrays               */
    double D;            /* coefficient of -lap in A_raw and L_raw (> 0)                   */
    usp_c128 sigma;      /* shift of L_raw (ignored when set_potential auto-scales)       */
    usp_c128 c;          /* scale c (ignored when set_potential auto-scales)              */
    void *stream;        /* cudaStream_t; NULL = legacy default stream                    */
    void *nccl_comm;     /* NULL = one GPU; else an ncclComm_t (usp_comm_init): the 3-D grid
                            is split into z-slabs over its ranks, one GPU per rank           */
    int virtual_ranks;   /* > 1 (with nccl_comm NULL): run the same slab decomposition with
                            this many slabs on ONE GPU, the transposes as device copies
                            (a test mode: every kernel, layout and index of the multi-GPU
                            path, no second GPU needed); 0 or 1 = off                        */
    int antisymmetric;   /* != 0: solve the antisymmetrised system of PAPER.md Eq. 9-10
                            (L100-128), E = [x; x'], A = c^-1 [[0, -A_raw^*], [A_raw, 0]]
                            with a REAL scale c, accretive for ANY A_raw (e.g. gain media,
                            where set_potential of the standard form fails); x' -> 0.
                            set_potential's canonical form: sigma = smallest-circle centre
                            of w, c = r / target_norm; no accretivity test.  2-D / 3-D
                            complex64, extents in [64, 1024], one GPU; 56 B per voxel of
                            workspace.  get_field returns x.                                */
    int tensor_diffusion; /* != 0: steady diffusion with a TENSOR D(r) in the first-order
                            (u, F) form of PAPER.md §3.2 Eqs. 16-18 (L199-227): d + 1 field
                            components, block-diagonal V; the medium is set with
                            usp_set_tensor_medium (mu_a and D); dtype must be USP_R32
                            (real mu_a, D, S; get_field returns u); 2-D / 3-D, extents in
                            [64, 1024], one GPU.                                             */
    /* Options.  Zero (a zero-initialised desc) selects the default behaviour
     * everywhere; no environment variable changes what a plan computes.      */
    int delta_form;       /* != 0: run the Delta-form recurrence of PAPER.md L613 from the
                             first iteration.  0: Algorithm 1 literally (x-form, L85-86,
                             8 fewer HBM bytes per voxel; s = S/c kept in the workspace)
                             while r_k >= r_switch, then the Delta-form (R-30).
                             The two are the same iteration in exact arithmetic.        */
    double r_switch;      /* x-form -> Delta-form threshold on r_k (0: 1e-2)                */
    int dense_source;     /* != 0: the x-form passes always read s densely.  0: when the
                             source lives on <= 64 x-lines, their x-transforms are added
                             after each x pass instead (R-31, exact up to fp32
                             rounding order).                                            */
    int separate_transposes; /* slab decomposition: != 0 selects NCCL all-to-all transposes
                             (device copies in virtual mode); 0: transposes fused into the
                             K_B / K_C stores over peer memory when every rank maps its
                             peers (else the all-to-alls, decided collectively).       */
    int complex_path;     /* != 0: float32 diffusion data on the complex64 path (widened on
                             the device); 0: the half-spectrum real path where supported
                             (3-D, medium USP_MEDIUM_W, R-26).                 */
    int launch_per_pass;  /* != 0: 2-D grids up to 512^2 launch one kernel per pass and
                             iteration; 0: one persistent cooperative launch per iterate
                             call (kernels_small.cu).                                    */
    int plane_chain;      /* != 0: on one GPU with nx = ny = 1024 (complex64, 3-D), each
                             iteration is the z pass plus ONE persistent kernel that runs
                             the y-inverse, x and y-forward passes plane by plane with the
                             plane's work array L2-resident (56
                             instead of 88 HBM B/voxel for the sparse-source x-form).  Same
                             arithmetic per element; only the residual's summation order
                             differs.  0: one sweep per FFT pass (K_B, K_C, K_D, K_A),
                             measured faster.                          */
    int test_hooks;       /* bit 0 (USP_HOOK_RANK_FINISH): on a one-rank communicator, reduce
                             the residual through the rank-ordered all-gather + k_finish
                             path of P > 1 plans (a test of that path on one GPU).  0 in
                             production.                                                  */
    int flat_work;        /* != 0: the z pass works in place on the chain buffer ([z][y][x],
                             16-column tiles of 128-byte rows).  0: on one GPU (3-D, ny and
                             nz in [64, 1024], not antisymmetric / tensor) the y-forward
                             pass writes a second chain buffer in the z-pair layout --
                             planes 2zp and 2zp+1 interleaved in 128-byte x blocks -- so
                             the z pass (K_C) moves 256-byte rows, and the y-inverse pass
                             reads it back (K_C 4.81 -> 4.58 ms at
                             1024^3, iteration -0.9 %; one more field of workspace).
                             Internal to the plan: fields are bit-identical either way.  */
} usp_plan_desc;

#define USP_HOOK_RANK_FINISH 1
#define USP_HOOK_WINDOW 2   /* one-rank communicator, workspace from usp_shared_alloc: register the
                               workspace as an NCCL window at usp_plan_set_workspace, write through
                               ncclGetPeerPointer's mapping and check the bytes through the plain
                               pointer, create the device communicator and run its LSA barrier
                               (the NEXT-1 transport's machinery on one GPU; tests only) */

/* How the slab decomposition's transposes move data (usp_transport). */
typedef enum {
    USP_TRANSPORT_NONE = 0,          /* one slab: no transposes                                  */
    USP_TRANSPORT_VIRTUAL = 1,       /* virtual slabs, fused into the K_B / K_C stores           */
    USP_TRANSPORT_VIRTUAL_COPY = 2,  /* virtual slabs, separate device-copy transposes            */
    USP_TRANSPORT_NCCL_WINDOW = 3,   /* fused stores into the peers' buffers through an NCCL 2.28
                                        window (ncclCommWindowRegister + ncclGetPeerPointer)     */
    USP_TRANSPORT_CUDA_IPC = 4,      /* fused stores into CUDA-IPC-mapped peer buffers            */
    USP_TRANSPORT_NCCL_ALLTOALL = 5  /* separate transposes: grouped ncclSend / ncclRecv          */
} usp_transport_kind;

/* Create a plan for the grid and problem described by *desc (copied).
 *
 * Slab decomposition (desc.nccl_comm or virtual_ranks > 1,
 * P slabs): a 3-D grid is split into P z-slabs of nz/P planes.  The x and y
 * FFT passes are slab-local; the z pass runs on y-slabs reached by an
 * all-to-all transpose (and back), and the residual norm is one all-gather
 * of P doubles summed in rank order, so every rank takes the same stop
 * decision.  The transposes are fused into the stores of
 * the y-forward and z passes (each row goes straight to the buffer of the
 * rank that needs it over NVLink: the peers' workspaces through an NCCL
 * window -- ncclCommWindowRegister + ncclGetPeerPointer, when the workspaces
 * come from usp_shared_alloc -- else CUDA-IPC mappings; resolved at
 * usp_plan_set_workspace, which is then collective), with a cross-rank
 * barrier after each; if any rank cannot map its peers (or P > 8, or
 * desc.separate_transposes) NCCL all-to-alls are used instead.  With nccl_comm, the arrays passed to
 * set_potential / set_source / get_field are the rank's slab
 * [nz/P][ny][nx] (usp_local_extent gives z0); every call is collective.
 * Requires P a power of two dividing ny and nz, ny and nz in [64, 2048].
 *
 * Errors: USP_ERR_ARG (NULL, ndim, D <= 0), USP_ERR_UNSUPPORTED (extent,
 * decomposition), USP_ERR_NCCL, USP_ERR_CUDA. */
usp_status usp_plan_create(const usp_plan_desc *desc, usp_plan_t *out);

/* Bytes of device workspace the plan needs: 4 complex64 fields
 * (x, Delta, B, work) = 32 bytes per local voxel; 6 (+ send and receive
 * buffers of the transposes) = 48 bytes per local voxel when P > 1; + one
 * more field for s on x-form plans (R-30) and for the z pass's plane-pair
 * buffer (desc.flat_work; the real path: half-spectrum rows instead). */
usp_status usp_plan_workspace_size(usp_plan_t plan, size_t *bytes);

/* Attach caller-owned device memory (>= workspace_size bytes, 256-B aligned).
 * Errors: USP_ERR_ARG (NULL, misaligned), USP_ERR_NOMEM (too small). */
usp_status usp_plan_set_workspace(usp_plan_t plan, void *dev, size_t bytes);

/* Local z-slab of this rank: first plane z0 and number of planes held
 * (z0 = 0, nz_local = nz on a single GPU and in virtual mode). */
usp_status usp_local_extent(usp_plan_t plan, int64_t *z0, int64_t *nz_local);

/* Set the medium (k^2 or w, see desc.medium / desc.dtype; [z][y][x]) and form
 * V = (w - sigma)/c and B = 1 - V on the device.
 * where: whether `medium` is a host or a device pointer.
 * target_norm > 0: canonical form (§2.2, §3.1): sigma, c are
 *   derived from the smallest circle enclosing the medium values (centre =
 *   bias, radius r), c = -i r/target_norm (K2) or r/target_norm (W), so that
 *   max|V| = target_norm; they replace desc.sigma / desc.c.
 * target_norm <= 0: use desc.sigma, desc.c as given.
 * Validation (Theorem 1 hypotheses, L58; Eq. 1): USP_ERR_NOT_CONTRACTIVE if
 * max|V| >= 1; USP_ERR_NOT_ACCRETIVE if Re(w/c) < -1e-6 |w/c| at some voxel
 * or D Re(c) < 0; USP_ERR_NONFINITE on NaN/Inf.  Invalidates the source. */
usp_status usp_set_potential(usp_plan_t plan, const void *medium, usp_where where,
                             double target_norm);

/* Medium of a tensor-diffusion plan (desc.tensor_diffusion; §3.2 Eqs. 16-18):
 * mu[n] = mu_a(r) (float32) and D[n][d(d+1)/2] the symmetric positive
 * definite diffusion tensor per voxel, packed (2-D: xx, xy, yy; 3-D: xx, xy,
 * xz, yy, yz, zz; [z][y][x] voxel order).  Canonical form (R-29):
 * mubar and Dbar^-1 = element-wise mid-ranges of mu and D^-1(r) (the centres
 * of the smallest circles of real values, L222-223), S = diag(s_u, s_F..)
 * with s_u, s_F the largest radii of the mu and D^-1 elements (the
 * equilibration), c = max_r max(|v_u|, ||V_F||_F) / target_norm so that
 * ||V|| <= target_norm.  usp_get_split reports sigma = mubar, c, centre =
 * (s_u, s_F), radius = radius of mu, max_abs_V.  Errors: USP_ERR_STATE (not a
 * tensor-diffusion plan), USP_ERR_NONFINITE (non-finite mu or a D that is not
 * positive definite), USP_ERR_ARG. */
usp_status usp_set_tensor_medium(usp_plan_t plan, const float *mu, const float *D, usp_where where,
                                 double target_norm);

/* Read back the split in use: sigma, c, smallest-circle centre and radius of
 * the medium values (0 if not auto-scaled), and max |V|. */
usp_status usp_get_split(usp_plan_t plan, usp_c128 *sigma, usp_c128 *c, usp_c128 *centre,
                         double *radius, double *max_abs_V);

/* Set the physical source S ([z][y][x], desc.dtype) and reset the state:
 * s = S/c, x_0 = 0, k = 0, Delta_0 = B (L+1)^-1 s, n0 = ||Delta_0|| (one FFT
 * round trip).  Requires set_potential first (USP_ERR_STATE). */
usp_status usp_set_source(usp_plan_t plan, const void *src, usp_where where);

/* Run at most n_max iterations of Algorithm 1 from the current state
 * (resumable; alpha may change between calls).  tol > 0: stop after the
 * first iteration k (0-based, counted from the last set_source) whose
 * r_k = ||Delta_k|| / n0 < tol; the returned field includes that update
 * (reading R-5).  tol <= 0: exactly n_max iterations.  Returns after the
 * termination decision (synchronises on the plan stream).
 * n_done: iterations done by this call; term: why it stopped.
 * Errors: USP_ERR_STATE (no source), USP_ERR_ARG (n_max < 0, alpha <= 0). */
usp_status usp_iterate(usp_plan_t plan, int64_t n_max, double alpha, double tol,
                       int64_t *n_done, usp_term *term);

/* Current residual: rel = ||Delta_k|| / n0 of the current x_k (after a
 * converged stop: of the last Delta the iteration used), abs_norm = n0 * rel,
 * k = iterations since set_source.  x-form plans may run one probe pass
 * (usp_iteration_form): collective with slab decomposition. */
usp_status usp_residual(usp_plan_t plan, double *rel, double *abs_norm, int64_t *k);

/* Copy r_0 .. r_{n-1} (fp64) into host[0..cap); *n = number available
 * (ring of the most recent 65536 iterations): n = k + 1 (r_k of the current
 * x_k included, computed on demand for x-form plans), except after a
 * converged stop of usp_iterate, where the final x_k's own residual is not
 * computed (reading R-5) and n = k (r_0 .. r_{k-1}, the last below tol). */
usp_status usp_residual_history(usp_plan_t plan, double *host, int64_t cap, int64_t *n);

/* Asynchronous input staging (pipelining a sequence of problems).
 * usp_staging_size: bytes of the caller-owned staging workspace: one medium
 * and one source of this plan (with_readback = 0), or those plus one field
 * for usp_get_field_async (with_readback != 0); each slot 256-byte aligned.
 * usp_plan_set_staging hands it over (it must outlive the plan; a staging
 * area of the smaller size supports usp_stage_inputs only).
 * usp_stage_inputs copies a medium and a source from host memory (pinned for
 * full speed; layouts and dtypes as usp_set_potential / usp_set_source) into
 * it on an internal copy stream and returns at once, so the copies overlap
 * whatever the plan stream is running (e.g. the iterations of the previous
 * problem).  The next usp_set_potential and usp_set_source called with
 * where = USP_STAGED (pointer argument ignored, may be NULL) make the plan
 * stream wait for those copies and use them.  Each slot is refilled only
 * after the plan stream has consumed it, and usp_stage_inputs refuses
 * (USP_ERR_STATE) while a staged medium has been taken by set_potential but
 * its source not yet by set_source, so a medium is never paired with the
 * next problem's source.  The host buffers must stay untouched until the
 * set_source(USP_STAGED) that consumes them has returned.  Not for
 * tensor-diffusion plans.  Errors: USP_ERR_STATE (no staging workspace /
 * nothing staged / source of the previous medium not consumed), USP_ERR_ARG,
 * USP_ERR_NOMEM (area too small), USP_ERR_UNSUPPORTED (tensor diffusion),
 * USP_ERR_CUDA. */
usp_status usp_staging_size(usp_plan_t plan, int with_readback, size_t *bytes);
usp_status usp_plan_set_staging(usp_plan_t plan, void *dev, size_t bytes);
usp_status usp_stage_inputs(usp_plan_t plan, const void *medium_host, const void *source_host);

/* Asynchronous result read-back (the staging workspace's third slot, see
 * usp_staging_size with with_readback != 0): usp_get_field_async snapshots
 * x_k into that slot on the plan stream and copies it to host memory `out`
 * (nz_local * ny * nx elements of desc.dtype) on a second copy stream,
 * returning at once -- the copy overlaps what the plan stream does next (the
 * next problem).  usp_wait_field blocks until that copy has landed; `out`
 * must not be read, and must stay allocated, before.  Errors: USP_ERR_STATE
 * (no staging workspace / no source), USP_ERR_NOMEM (staging area sized
 * without the read-back slot), USP_ERR_UNSUPPORTED (tensor-diffusion plans;
 * float32 fields on the complex path, desc.complex_path), USP_ERR_ARG,
 * USP_ERR_CUDA. */
usp_status usp_get_field_async(usp_plan_t plan, void *out_host);
usp_status usp_wait_field(usp_plan_t plan);

/* Copy the current iterate x_k into `out` ([z][y][x], desc.dtype). */
usp_status usp_get_field(usp_plan_t plan, void *out, usp_where where);

/* BiCGSTAB on the preconditioned system (PAPER.md
 * Eq. 5 L73-76 and Table 1b, van der Vorst 1992):
 *     M x = b,   M = B [1 - (L+1)^-1 B]  (Gamma^-1 A with alpha = 1; the
 *     iterates do not depend on alpha, R-25),  b = B (L+1)^-1 s,
 * x_0 = 0, shadow residual rhat = r_0 = b.  A pass is two applications of M
 * (the fixed-point path's FFT passes).  Stops when ||s||/||b|| < tol after
 * the half step (then x += a p) or ||r||/||b|| < tol after the full step
 * (r = b - M x, the fixed-point path's Delta, reading R-4); tol <= 0 runs
 * exactly n_max passes.  n_done = passes; usp_residual / _history report
 * ||r_k|| / ||b|| per pass.  Needs a Krylov workspace (5 complex64 fields:
 * rhat, p, v, s, t; 40 bytes per voxel, caller-owned, 256-B aligned) and
 * the state right after usp_set_source (not resumable).  2-D / 3-D
 * complex64 plans on one GPU (incl. virtual slabs).
 * Errors: USP_ERR_STATE, USP_ERR_ARG, USP_ERR_UNSUPPORTED, USP_ERR_NOMEM;
 * term = USP_DIVERGED also on a BiCGSTAB breakdown (rho, (rhat, v) or (t, t)
 * exactly 0). */
usp_status usp_krylov_workspace_size(usp_plan_t plan, size_t *bytes);
usp_status usp_krylov_set_workspace(usp_plan_t plan, void *dev, size_t bytes);
usp_status usp_bicgstab(usp_plan_t plan, int64_t n_max, double tol, int64_t *n_done, usp_term *term);

/* Restarted GMRES(m) on the same system M x = b (
 * Table 1b's GMRES5 / GMRES20 columns; Saad & Schultz
 * 1986), reading R-28: x_0 = 0, restart every m Arnoldi steps,
 * classical Gram-Schmidt applied twice (CGS2) by fused multi-dot / multi-axpy
 * kernels over blocks of 8 basis vectors, Givens rotations and the small
 * least-squares solve on the host in fp64.  Stops when the residual
 * estimate |g_{j+1}| / ||b|| < tol (then x is updated) or after n_max
 * Arnoldi steps; n_done = Arnoldi steps; the residual history is the estimate
 * per step.  Workspace: b and the basis U_0..U_m (m + 2 complex64 fields,
 * caller-owned, 256-B aligned); 2-D / 3-D complex64, also slab-decomposed
 * (the inner products are all-gathered and summed in rank order, so every
 * rank takes the same decisions); starts right after usp_set_source.
 * Errors as usp_bicgstab. */
usp_status usp_gmres_workspace_size(usp_plan_t plan, int m, size_t *bytes);
usp_status usp_gmres_set_workspace(usp_plan_t plan, int m, void *dev, size_t bytes);
usp_status usp_gmres(usp_plan_t plan, int64_t n_max, double tol, int64_t *n_done, usp_term *term);

/* Kernel timing (CUDA events on the plan stream, per kernel class) for the
 * roofline report.  enable != 0 starts accumulating; usp_profile_read copies
 * up to cap entries of (name, total ms, launches) for the kernel classes. */
usp_status usp_profile_enable(usp_plan_t plan, int enable);
usp_status usp_profile_read(usp_plan_t plan, int cap, char (*names)[32], double *ms,
                            int64_t *launches, int *n);

/* Number of kernel launches the library issued since plan creation. */
usp_status usp_launch_count(usp_plan_t plan, int64_t *launches);

/* Algebraic form of the iteration (reading R-30).  xform = 1: the
 * plan runs Algorithm 1 literally (x-form: 8 fewer HBM bytes per
 * voxel and iteration; s = S/c kept in the workspace) while the last
 * residual is >= r_switch (desc.r_switch, default 1e-2; desc.delta_form
 * disables), then the Delta-form recurrence (exact
 * down to fp32 rounding near convergence).  form: 0 = Delta-form now,
 * 1 = x-form now.  source_lines > 0: the source lives on that many x-lines
 * (<= 64) and the x-form passes never read s (reading R-31: the x-transformed
 * source lines are added after each x pass); 0: s is read densely
 * (desc.dense_source, or a source on more lines).  After
 * x-form iterations, r_k and Delta_k of the current
 * x_k are computed on demand by usp_residual / usp_residual_history (one
 * probe pass: x unchanged); those two calls are therefore collective over
 * the ranks of a slab-decomposed plan.  Errors: USP_ERR_ARG. */
usp_status usp_iteration_form(usp_plan_t plan, int *xform, int *form, double *r_switch, int *source_lines);

/* Workspace memory for slab-decomposed plans over a communicator: ncclMemAlloc
 * (symmetric memory NCCL can register as a window, so the fused transposes
 * reach the peers' buffers through ncclGetPeerPointer -- SURVEY.md §8(f)
 * NEXT-1) when libnccl.so.2 (>= 2.28) provides it, else cudaMalloc.  The
 * caller owns it and frees it with usp_shared_free after usp_plan_destroy.
 * Errors: USP_ERR_ARG, USP_ERR_NOMEM. */
usp_status usp_shared_alloc(size_t bytes, void **ptr);
usp_status usp_shared_free(void *ptr);

/* *kind = the usp_transport_kind the plan's transposes use (decided at
 * usp_plan_set_workspace; collectively for NCCL plans).  Errors: USP_ERR_ARG. */
usp_status usp_transport(usp_plan_t plan, int *kind);

/* *zpair = 1 if the plan's z pass runs on the z-pair chain buffer
 * (desc.flat_work), else 0.  Diagnostic; no device work.  Errors: USP_ERR_ARG. */
usp_status usp_work_layout(usp_plan_t plan, int *zpair);

/* NCCL communicator for the slab decomposition (one process per GPU).
 * Rank 0 calls usp_comm_unique_id and broadcasts the 128 bytes (e.g. with
 * torch.distributed); every rank then calls usp_comm_init with the same id,
 * the rank count and its rank (collective; the current CUDA device is the
 * rank's GPU).  libnccl.so.2 is opened at run time (USP_NCCL_LIB overrides
 * the path).  Errors: USP_ERR_ARG, USP_ERR_NCCL. */
usp_status usp_comm_unique_id(unsigned char id[128]);
usp_status usp_comm_init(const unsigned char id[128], int nranks, int rank, void **comm);
usp_status usp_comm_destroy(void *comm);

/* Release the plan (not the caller's workspace).  NULL is a no-op. */
void usp_plan_destroy(usp_plan_t plan);

/* Thread-local message describing the last error ("" if none). */
const char *usp_last_error(void);

/* "major.minor sm_100a" */
const char *usp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* USP_H */
