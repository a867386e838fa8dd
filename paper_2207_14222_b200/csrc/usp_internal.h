// usp_internal.h -- structures shared by the kernels (kernels.cu) and the
// plan/driver (usp_api.cu).  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace usp {

// Iteration status kept on the device so launched batches can stop
// themselves without a host round trip.
enum : int {
    ST_RUNNING = 0,      // iterate: full iteration (chain + update)
    ST_STOP_PENDING = 1, // r_k < tol: the next iteration only applies x += alpha Delta_k
    ST_DONE_CONV = 2,    // converged, final update applied
    ST_DIVERGED = 3,     // non-finite or r > 1e6
    ST_NO_SOURCE = 4
};

struct IterState {
    double alpha;        // step size (Algorithm 1 line 4)
    double tol;          // stop threshold (<= 0: none)
    double n0;           // ||Delta_0|| = ||B (L+1)^-1 s||  (reading R-4)
    double r;            // r_k = ||Delta_k|| / n0 of the current Delta_k
    long long k;         // iterations done since set_source (x_k is current)
    long long kmax;      // absolute iteration limit of the running iterate call
    int status;
    unsigned int counter;  // last-block-done counter (reset by the last block)
    int err;               // pipeline watchdog: non-zero = a kernel gave up waiting (see tma.cuh)
    int err_info;
    // Algebraic form of the x pass (reading R-30): FORM_DELTA = Delta-form
    // recurrence; FORM_X = Algorithm 1 literally (needs s,
    // 8 fewer bytes per voxel); FORM_PROBE = one pass that computes Delta_k
    // of the x-form state without updating x (end of an iterate call).  An
    // x-form pass whose previous residual is below r_sw converts the state
    // to the Delta-form instead (see xform_act).
    int form;
    int xform;             // the plan runs the x-form while r >= r_sw (set at set_source)
    double r_sw;
    int add_s;             // sparse source: the last x pass formed u = B x (+ s still to add)
};

enum : int { FORM_DELTA = 0, FORM_X = 1, FORM_PROBE = 2 };
// what an x-pass launch does, decided from the state every CTA reads at its start
enum : int { ACT_DELTA = 0, ACT_X = 1, ACT_PROBE = 2, ACT_TO_DELTA = 3 };

struct Red {             // reduction scratch (device)
    double *partials;    // one per CTA of the reducing kernel
    double *hist;        // residual ring
    int hist_cap;
    double *local_sum;   // slab-decomposed: the x pass stores its total here (else nullptr)
};

// Fourier multiplier data of (L+1)^-1 = F^-1 [c/(D|p|^2 + sigma + c)] F (Eq. 12),
// with the inverse DFT's 1/N_vox folded into the numerator.
struct MulParams {
    float2 cn;           // c / N_vox
    float2 sc;           // sigma + c
    float D;
    float sqrtD;         // sqrt(D) (the z pass folds it into the line frequency)
    float kx, ky, kz;    // 2 pi / (n_a h_a): p_a = k_a * m_a
    int nx, ny, nz;
    int rowc;            // columns per row of the spectrum array (nx; nx/2 + 16 on the real path)
};

// ------------------------------------------------- chain-buffer layout --
// z-pair layout (default; desc.flat_work disables; one-GPU 3-D plans with
// ny, nz in [64, 1024]): the z pass runs on a second chain
// buffer `work2` in which planes 2zp and 2zp + 1 are interleaved in
// 16-element (128-byte) blocks of the row (rp = nx, or nx/2 + 16 on the
// real path),
//   work2[((zp * ny + y) * (rp / 16) + x / 16) * 32 + (z % 2) * 16 + x % 16],
// so its 16-column tiles read and write 256-byte rows (the z pattern's DRAM
// efficiency depends on the row width: tools/micro/zwrite.cu, zpairlay.cu).
// K_B writes work -> work2 in that layout, K_D reads work2 through the
// [nz/2][ny][2 rp] view and writes work back in [z][y][rp]; the x pass
// never sees it.

// ---------------------------------------------------------------- x pass --
enum XMode : int { X_SRC_FWD = 0, X_SRC_EPI = 1, X_ITER = 2 };

struct XParams {
    float2 *work;        // chain buffer (complex64, [z][y][x])
    float2 *delta;       // Delta_k
    float2 *x;           // x_k (also the staging area of the raw source S)
    const float2 *B;     // B = 1 - V
    const float2 *tw;    // four-step twiddles for nx (real path: for nx/2)
    const float2 *twr;   // real path: W_nx^k, k < nx/2 (split/merge of the half-length FFT)
    long long nlines;    // ny * nz (local)
    int src_real;        // staged source is float32 (else complex64)
    float2 inv_c;        // 1/c (s = S/c)
    IterState *st;
    Red red;
    float2 *s;           // x-form plans: s = S / c (else nullptr)
    // sparse source (R-31): the x pass forms u = B x and k_sadd adds the
    // x-transformed source lines afterwards; X_SRC_FWD flags the source lines
    unsigned char *s_flag;   // per x-line: s != 0 (written by X_SRC_FWD when non-null)
    int s_sparse;            // X_ITER: do not read s (its x-transform is added by k_sadd)
};

// sparse source lines (R-31): line l = list[i] of the local grid gets comp[i*N .. +N) added
struct SAddParams {
    float2 *work;
    const float2 *comp;
    const int *list;
    int count;
    int n;               // line length (row pitch of work)
    IterState *st;
};

// ------------------------------------------------------- BiCGSTAB (NEXT-2) --
enum KMode : int { K_PFWD = 0, K_VINV = 1, K_SFWD = 2, K_TINV = 3, K_OFWD = 4, K_OINV = 5 };

// GMRES(m) Gram-Schmidt blocks (kernels_krylov.cu k_gs)
enum GSMode : int { GS_DOT = 0, GS_AXPY = 1 };
struct GSParams {
    const float2 *U[8];  // basis block
    float2 c[8];         // GS_AXPY coefficients
    float2 scale;        // GS_AXPY: z <- scale (z - sum c_j U_j)
    float2 *z;
    long long n;
    double *partials;    // per CTA: 2 NB + 1 (GS_DOT) or 1 (GS_AXPY) doubles
};

struct KState {          // BiCGSTAB scalars (fp64, device)
    double2 rho, alpha, omega, beta;
    double nb;           // ||b|| = ||B (L+1)^-1 s|| (= n0 of the fixed-point iteration)
    double res_s;        // ||s|| / ||b|| of the current pass (half-step test)
    int breakdown;       // rho, (rhat, v) or (t, t) became exactly 0
};

struct KParams {
    float2 *work, *x, *r, *rh, *p, *v, *s, *t;
    const float2 *B;
    const float2 *tw;    // four-step twiddles for nx
    long long nlines;    // ny * nz
    long long nvox;
    IterState *st;
    KState *ks;
    double *partials;    // >= 3 doubles per CTA
    double *hist;
    int hist_cap;
};

// ---------------------------------------------------------- strided pass --
constexpr int kMaxPeers = 8;   // ranks of a fused (peer-memory) slab decomposition
enum SMode : int { S_FWD = 0, S_INV = 1, S_FWD_MUL_INV = 2 };

struct SParams {
    float2 *data;        // field the pass reads (in place unless dst differs)
    float2 *dst;         // where results are stored (== data for in-place passes)
    const float2 *tw;    // four-step twiddles for the line length
    long long stride;    // elements between consecutive line points
    long long ncols;     // columns per outer slab (contiguous)
    long long nouter;    // outer slabs
    long long ostride;   // elements between outer slabs
    int line_axis;       // 1 = y (2-D, columns = x), 2 = z (3-D, columns = (y, x))
    int check_state;     // 0: always run; 1: skip unless status == RUNNING && k < kmax
    MulParams mp;
    IterState *st;
    // slab decomposition (k_stile only; P = 1: natural layout everywhere)
    int map_rank;        // tensor map rank: 2, 3 (y pass, 3-D) or 5 (send layout)
    int send_layout;     // S_FWD: store into the send layout [r][q][z_loc][y_loc][x]
    int P;               // slabs per rank group
    int nz_loc;          // z planes per slab
    int nyl_lg;          // log2(ny / P)
    long long y0;        // global y of this rank's y block (z pass multiplier)
    int col0;            // x-chunked transposes: column offset of the load map's coordinates (K_B)
    int x0;              // x-chunked transposes: global x of the chunk's column 0 (z pass multiplier;
                         // mp.rowc is then the chunk width)
    int zpair;           // K_C on the z-pair buffer: a tile row is 32 columns (16 x of planes
                         // 2zp, 2zp + 1), rows = plane pairs, stride = pair-row pitch
    int pair_dst;        // K_B: store plane o into the z-pair buffer (stride = 2 nx, ostride =
                         // 2 nx ny per plane pair)
    int pair_src;        // K_D: load plane o through the map of the [nz/2][ny][2 nx] view
    int tma_store;       // k_stile: store the upper half of each tile (rows >= N/2; all rows for
                         // N <= 256) through the exchange buffer with tensor-map stores on the
                         // load map (in-place passes whose map describes dst only)
    // transposes fused into the stores (slab decomposition, peer memory):
    // 1 = K_B stores into the ranks' receive buffers, 2 = K_C stores into the
    // ranks' send buffers; peer[q] = rank q's buffer (this GPU's own for q = rank,
    // CUDA-IPC-mapped peer memory over NVLink for the others, or the virtual
    // ranks' regions of one buffer)
    int peer_mode;
    int rank0;           // rank of this plan's first slab / y block (NCCL: the rank; virtual: 0)
    long long bk;        // elements per transpose block (nz_loc * ny_loc * row pitch)
    float2 *peer[kMaxPeers];
};

// ------------------------------------------- plane-chained pass (NEXT-4) --
// K_D -> K_A -> K_B of one iteration in one persistent kernel, plane by
// plane, `work` L2-resident in between (kernels_plane.cu); nx = ny = kPlaneN.
constexpr int kPlaneN = 1024;
struct PParams {
    float2 *work, *x, *delta;
    const float2 *B;
    const float2 *s;             // x-form plans: s = S / c (dense); else nullptr
    const float2 *tw;            // four-step twiddles of kPlaneN (x and y)
    long long nz;                // planes
    int s_sparse;                // sparse source (R-31): add s_comp lines instead of reading s
    const int *s_list;
    const float2 *s_comp;
    int s_count;
    unsigned long long *ctr;     // y unit counter (reset by the last CTA)
    unsigned *d_done, *a_done;   // per plane: finished y-inverse tiles / x lines
    double *upart;               // per x line: residual partial (nz * nx)
    int ny_ctas;                 // CTAs in the y role (the rest run the x role)
    IterState *st;
    Red red;
};
cudaError_t launch_plane(const CUtensorMap &mapy, const PParams &p, int grid, cudaStream_t s, bool lean,
                         bool expect_x);

// ------------------------------------------------------------------ 1-D --
enum OneMode : int { O_SETUP = 0, O_ITER = 1 };
struct OneParams {
    float2 *delta, *x;
    const float2 *B;
    const float2 *tw;
    int src_real;
    float2 inv_c;
    MulParams mp;
    IterState *st;
    Red red;
};

// ------------------------------------------- antisymmetrised system (NEXT-3) --
struct AParams {
    float2 *work, *delta, *x;  // two components each, component-major (component 2 at + nvox)
    const float2 *v;           // v = (w - sigma)/c
    const float2 *tw;          // four-step twiddles for nx
    long long nlines;          // ny * nz
    long long nvox;            // voxels per component
    float inv_c;               // 1/c (c real)
    float2 sigma;
    float inv_n;               // 1 / N_vox (the inverse DFT's normalisation)
    MulParams mp;
    IterState *st;
    Red red;
};

// ------------------------------------------- tensor diffusion (NEXT-3) --
struct TDParams {
    int d;                       // 2 or 3 (components d + 1: u, F_x, F_y[, F_z])
    long long n;                 // voxels
    float2 *work, *delta, *x;    // (d + 1) components each, component-major
    const float *mu, *Dpk;       // setup inputs: mu_a, D packed symmetric (xx, xy, [xz,] yy[, yz, zz])
    float *dinv;                 // per-voxel D^-1 packed
    float *vu, *vf;              // V per voxel: u block, flux block (packed)
    float mubar, inv_cu, inv_cf; // 1/(c s_u), 1/(c s_F)
    float dbar[6];               // Dbar^-1 packed
    float a, qs, inv_n;          // symbol: a = mubar/(c s_u) + 1, q = p qs, 1/N_vox
    float dm_inv[9];             // (Dbar^-1/(c s_F) + I)^-1, row-major 3x3
    const float *Sraw;           // staged raw source
    float s_scale;               // 1/(c sqrt(s_u))
    float *red;                  // setup reductions: 16 floats per CTA
    MulParams mp;
    const float2 *twx;           // x-line twiddles (the fused x pass)
    IterState *st;
    Red red_d;
};

// ------------------------------------------------- persistent 2-D solve --
struct S2Params {
    float2 *work, *delta, *x;
    const float2 *B;
    const float2 *twx, *twy;   // four-step twiddles for nx, ny
    MulParams mp;
    IterState *st;
    Red red;                   // hist
    double *partials;          // 2 x gridDim doubles (double-buffered per iteration)
    unsigned *bar_count;       // grid barrier (zeroed at plan creation)
    unsigned *bar_gen;
};

// --------------------------------------------------------------- setup --
struct PotParams {
    const void *medium;  // staged medium (device)
    int medium_real;     // float32 (else complex64)
    int medium_is_k2;    // w = -k^2 (else w = medium)
    float2 *B;           // out: B = 1 - V
    long long n;
    double sig_re, sig_im, c_re, c_im;
    // outputs (atomics)
    unsigned int *max_absV_bits;  // float bits of max |V| (non-negative -> int order)
    unsigned int *n_nonaccretive;
    unsigned int *n_nonfinite;
    int b_real;          // store B as float32 (real path; V is real there)
    int store_v;         // antisymmetrised system: store v = V instead of B, no accretivity test
};

struct FarParams {       // farthest medium value from a centre (smallest circle)
    const void *medium;
    int medium_real;
    long long n;
    double cre, cim;
    double *best_d2;     // per CTA
    long long *best_idx; // per CTA
};

// antisymmetrised system (kernels_anti.cu)
cudaError_t launch_anti_x(int N, XMode mode, const AParams &p, int grid, cudaStream_t s);
cudaError_t launch_anti_mul(const AParams &p, int check_state, int grid, cudaStream_t s);
int anti_lines_per_cta(int N);
cudaError_t launch_anti_pipe(int N, const AParams &p, int grid, cudaStream_t s);   // the iterations' x pass
int anti_pipe_units(int N);                                                        // lines per warp unit

// tensor diffusion (kernels_tdiff.cu)
cudaError_t launch_xfft(int N, bool inv, float2 *data, const float2 *tw, long long nlines, int grid, cudaStream_t s);
cudaError_t launch_tdiff_pot(const TDParams &p, int mode, int grid, cudaStream_t s);
cudaError_t launch_tdiff_mul(const TDParams &p, int check_state, int grid, cudaStream_t s);
cudaError_t launch_tdiff_pipe(int N, const TDParams &p, int grid, cudaStream_t s);   // fused x pass; Invalid if the stage does not fit
int tdiff_pipe_units(int N, int d);                                                  // 0: falls back to k_xfft + k_tdiff_upd
cudaError_t launch_tdiff_upd(XMode mode, const TDParams &p, int grid, cudaStream_t s);
cudaError_t launch_tdiff_out(const float2 *E0, float *out, float scale, long long n, int grid, cudaStream_t s);

// persistent 2-D solve (kernels_small.cu)
bool solve2d_supported(long long nx, long long ny);
cudaError_t launch_solve2d(int nx, int ny, const S2Params &p, int nsm, cudaStream_t s);

// BiCGSTAB (kernels_krylov.cu)
cudaError_t launch_xop(int N, KMode mode, const KParams &p, int grid, cudaStream_t s);
cudaError_t launch_kupd(const KParams &p, int grid, cudaStream_t s);
constexpr int kGsCtasPerSm = 3;   // k_gs: __launch_bounds__(256, 3), grid = 3 x SMs
cudaError_t launch_gs(int mode, int nb, const GSParams &p, int grid, cudaStream_t s);

// real path (kernels_real.cu)
cudaError_t launch_xpass_real(int N, XMode mode, const XParams &p, int grid, cudaStream_t s);
bool xreal_supported(long long n);
int xreal_row_pitch(int N);
int xreal_lines_per_unit(int N);

// launchers (kernels.cu); all return cudaGetLastError()
cudaError_t launch_strided(int N, SMode mode, const SParams &p, int grid, cudaStream_t s);   // N = 16, 32
cudaError_t launch_solve1d(int N, OneMode mode, const OneParams &p, cudaStream_t s);
cudaError_t launch_potential(const PotParams &p, int grid, cudaStream_t s);
cudaError_t launch_farthest(const FarParams &p, int grid, cudaStream_t s);
int farthest_grid(int grid);   // grid clamped to the CTAs resident at once (one partial per CTA)
cudaError_t launch_finish(IterState *st, const double *sums, int P, int src_epi, const Red &red, cudaStream_t s);
cudaError_t launch_set_state(IterState *st, double alpha, double tol, long long kmax, cudaStream_t s);
// small host -> device writes as kernel arguments (no copy engine, no pageable-memory copy)
struct Blob { unsigned char b[512]; };
cudaError_t launch_put_bytes(void *dst, const void *src, size_t n, cudaStream_t s);
cudaError_t launch_put_state(IterState *st, const IterState &h, cudaStream_t s);
cudaError_t launch_set_form(IterState *st, int form, cudaStream_t s);
cudaError_t launch_copy_bytes(void *dst, const void *src, size_t n, int grid, cudaStream_t s);
cudaError_t launch_sparse_count(const unsigned char *flag, long long nlines, unsigned *count, cudaStream_t s);
cudaError_t launch_sparse_gather(const unsigned char *flag, long long nlines, const float2 *work, int n, int *list,
                                 float2 *comp, unsigned *count, cudaStream_t s);
cudaError_t launch_sparse_add(const SAddParams &p, cudaStream_t s);

// TMA-pipelined variants (kernels_pipe.cu)
cudaError_t launch_xpass_pipe(int N, XMode mode, const XParams &p, int grid, cudaStream_t s, bool lean = false,
                              bool expect_x = false);

// TMA-prefetched 16-column strided passes (kernels_stile.cu)
// smap: the map the half-tile tensor-map stores (SParams::tma_store) write through
// (the load map for in-place passes)
cudaError_t launch_stile(int N, SMode mode, const CUtensorMap &map, const CUtensorMap &smap, const SParams &p, int grid,
                         cudaStream_t s);
bool stile_supported(long long n);
int stile_cols(int N);
int stile_box(int N);
int stile_ctas_per_sm(int N);

bool supported_n(long long n);

}  // namespace usp
