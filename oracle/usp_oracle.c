/*
 * usp_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path
 * of the universal split preconditioner (Vettenburg & Vellekoop,
 * arXiv 2207.14222, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA product in
 * paper_2207_14222_b200/ and includes nothing from it.
 *
 * Precision: complex128 / float64 throughout (the paper fixes no precision
 * for the method; its own runs were fp32).
 *
 * Unified form (reading R-1):
 *     A_raw = -D lap + w(r),   L_raw = -D lap + sigma,   V_raw = w - sigma
 *     A = A_raw / c,  L = L_raw / c,  V = V_raw / c,  s = S_raw / c
 * (§2.2 "divide the original problem by a complex scalar c").
 * Helmholtz (Eq. 8) is D = 1, w = -k^2, sigma = -kbar^2,
 * c = -i r / 0.95 (the paper's c = i r/0.95 with the equation times -1).
 *
 * Functions (each cites the passage it follows):
 *   orc_fft1d     radix-2 DFT, forward e^{-2 pi i jk/N} unnormalised,
 *                 inverse e^{+...} with 1/N (reading R-8).
 *   orc_fftn      n-D DFT = 1-D DFT along every axis (PAPER.md L171:
 *                 "the Fourier transform over all spatial dimensions").
 *   orc_apply_Linv  (L+1)^-1 = F^-1 c/(D|p|^2 + sigma + c) F   (Eq. 12,
 *                 PAPER.md L168-172; p = 2 pi fftfreq(N, h), reading R-7).
 *   orc_setup     V = (w - sigma)/c, B = 1 - V, s = S/c.
 *   orc_fixed_point  Algorithm 1 literally (x-form), or
 *                 the Neumann recurrence Delta_i = (1 - Gamma^-1 A) Delta_{i-1}
 *                 (the Delta-form) for the R-17 cross-check.
 *   orc_mec       smallest enclosing circle ("smallest circle
 *                 problem"), Welzl's randomised incremental algorithm.
 *   orc_fixed_point_anti  Algorithm 1 on the antisymmetrised system of Eq. 9-10
 *                 (PAPER.md L100-128): E = [x, x'], A = c^-1 [[0, -A_raw*], [A_raw, 0]],
 *                 real c, for problems whose numerical range is not confined
 *                 to a half plane (e.g. gain media).
 *   orc_fixed_point_tdiff  Algorithm 1 on the first-order (u, F) form of
 *                 steady diffusion with a tensor D (§3.2 Eqs. 16-18,
 *                 L199-227): d + 1 components, block-diagonal V.
 *   orc_gmres     restarted GMRES(m) (Saad & Schultz 1986; Table 1b's GMRES5 /
 *                 GMRES20 columns) on the same system.
 *   orc_bicgstab  BiCGSTAB [van der Vorst 1992, cited PAPER.md L384] on the
 *                 preconditioned system Gamma^-1 A x = Gamma^-1 s with
 *                 Gamma^-1 A = alpha B[1 - (L+1)^-1 B] (Eq. 5, PAPER.md
 *                 L73-76); the "BiCGSTAB" column of Table 1b (L305-311).
 *
 * Error behaviour: every entry point returns 0 on success, a negative code on
 * bad arguments (-1 non-power-of-two extent, -2 bad ndim/size, -3 alloc).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static const double ORC_PI = 3.14159265358979323846264338327950288;

static int is_pow2(long n) { return n >= 1 && (n & (n - 1)) == 0; }

/* ---------------------------------------------------------------- FFT -- */

/* In-place iterative radix-2 decimation-in-time DFT of length n (power of 2).
 * tw[k] = exp(-2 pi i k / n), k < n/2 (forward); the inverse conjugates and
 * divides by n at the end.  Textbook Cooley-Tukey: bit-reverse, then log2 n
 * butterfly sweeps. */
static void fft1d_with_table(cplx *a, long n, const cplx *tw, int inverse) {
    if (n <= 1) return;
    for (long i = 1, j = 0; i < n; ++i) {           /* bit reversal */
        long bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { cplx t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (long len = 2; len <= n; len <<= 1) {
        long half = len >> 1, step = n / len;
        for (long i = 0; i < n; i += len) {
            for (long j = 0; j < half; ++j) {
                cplx w = tw[j * step];
                if (inverse) w = conj(w);
                cplx u = a[i + j];
                cplx v = a[i + j + half] * w;
                a[i + j] = u + v;
                a[i + j + half] = u - v;
            }
        }
    }
    if (inverse) {
        double inv = 1.0 / (double)n;
        for (long i = 0; i < n; ++i) a[i] *= inv;
    }
}

static cplx *make_twiddles(long n) {
    long m = n / 2 > 0 ? n / 2 : 1;
    cplx *tw = (cplx *)malloc(sizeof(cplx) * (size_t)m);
    if (!tw) return NULL;
    for (long k = 0; k < m; ++k) {
        double ang = -2.0 * ORC_PI * (double)k / (double)n;
        tw[k] = cos(ang) + I * sin(ang);
    }
    return tw;
}

int orc_fft1d(double *data, long n, int inverse) {
    if (!is_pow2(n)) return -1;
    cplx *tw = make_twiddles(n);
    if (!tw) return -3;
    fft1d_with_table((cplx *)data, n, tw, inverse);
    free(tw);
    return 0;
}

/* n-D DFT of a C-ordered array (dims[ndim-1] contiguous): a 1-D DFT along
 * each axis in turn.  Lines are independent, so they are spread over OpenMP
 * threads.  Each thread copies a group of up to ORC_GROUP lines that are
 * adjacent in memory (neighbouring columns of a strided axis) into its own
 * scratch buffer, transforms each line on its own with fft1d_with_table, and
 * copies them back: the per-line arithmetic is the plain DFT above, the
 * grouping only makes the strided copies use whole cache lines. */
#define ORC_GROUP 8
int orc_fftn(double *data, int ndim, const long *dims, int inverse) {
    if (ndim < 1 || ndim > 3) return -2;
    long total = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        total *= dims[a];
    }
    cplx *x = (cplx *)data;
    for (int a = 0; a < ndim; ++a) {
        long n = dims[a];
        if (n == 1) continue;
        long stride = 1;
        for (int b = a + 1; b < ndim; ++b) stride *= dims[b];
        long outer = total / (n * stride);
        long grp = stride < ORC_GROUP ? stride : ORC_GROUP;   /* stride, ORC_GROUP: powers of 2 */
        long ngroups = outer * (stride / grp);
        cplx *tw = make_twiddles(n);
        if (!tw) return -3;
        int err = 0;
#pragma omp parallel
        {
            cplx *lines = (cplx *)malloc(sizeof(cplx) * (size_t)(n * grp));
            if (!lines) {
#pragma omp atomic write
                err = 1;
            } else {
#pragma omp for schedule(static)
                for (long gi = 0; gi < ngroups; ++gi) {
                    long o = gi / (stride / grp), i0 = (gi % (stride / grp)) * grp;
                    cplx *base = x + o * n * stride + i0;
                    for (long t = 0; t < n; ++t)
                        for (long b = 0; b < grp; ++b) lines[b * n + t] = base[t * stride + b];
                    for (long b = 0; b < grp; ++b) fft1d_with_table(lines + b * n, n, tw, inverse);
                    for (long t = 0; t < n; ++t)
                        for (long b = 0; b < grp; ++b) base[t * stride + b] = lines[b * n + t];
                }
                free(lines);
            }
        }
        free(tw);
        if (err) return -3;
    }
    return 0;
}

/* ------------------------------------------------------- (L + 1)^{-1} -- */

/* Angular frequency p_a(m) = 2 pi fftfreq(n, h)[m] (reading R-7). */
static double freq(long m, long n, double h) {
    long mm = (m < (n + 1) / 2) ? m : m - n;   /* numpy.fft.fftfreq ordering */
    if (n % 2 == 0 && m == n / 2) mm = -n / 2;
    return 2.0 * ORC_PI * (double)mm / ((double)n * h);
}

/* g(p) = c / (D |p|^2 + sigma + c): the Fourier multiplier of (L+1)^-1 in the
 * unified form; Eq. 12 L170 is the Helmholtz case
 * c/(-|p|^2 + kbar^2 + c) with (D, sigma, c) -> (1, -kbar^2, -c). */
static cplx g_of(double p2, double D, cplx sigma, cplx c) {
    return c / (D * p2 + sigma + c);
}

/* u <- (L+1)^{-1} u = F^{-1} g F u   (Eq. 12). */
int orc_apply_Linv(double *u, int ndim, const long *dims, const double *h, double D,
                   double sig_re, double sig_im, double c_re, double c_im) {
    int rc = orc_fftn(u, ndim, dims, 0);
    if (rc) return rc;
    cplx sigma = sig_re + I * sig_im, c = c_re + I * c_im;
    long nx = dims[ndim - 1];
    long ny = ndim >= 2 ? dims[ndim - 2] : 1;
    long nz = ndim >= 3 ? dims[ndim - 3] : 1;
    double hx = h[ndim - 1];
    double hy = ndim >= 2 ? h[ndim - 2] : 1.0;
    double hz = ndim >= 3 ? h[ndim - 3] : 1.0;
    cplx *x = (cplx *)u;
#pragma omp parallel for schedule(static)
    for (long l = 0; l < nz; ++l) {
        double pz = ndim >= 3 ? freq(l, nz, hz) : 0.0;
        for (long j = 0; j < ny; ++j) {
            double py = ndim >= 2 ? freq(j, ny, hy) : 0.0;
            for (long i = 0; i < nx; ++i) {
                double px = freq(i, nx, hx);
                double p2 = px * px + py * py + pz * pz;
                x[(l * ny + j) * nx + i] *= g_of(p2, D, sigma, c);
            }
        }
    }
    return orc_fftn(u, ndim, dims, 1);
}

/* ----------------------------------------------------------- splitting -- */

/* V = (w - sigma)/c, B = 1 - V, s = S/c   ("B := 1 - V",
 * L92-97 "A := c^-1 A_raw ... b := c^-1 b_raw", V := A - L). */
int orc_setup(const double *w, const double *S, long n, double sig_re, double sig_im,
              double c_re, double c_im, double *V_out, double *B_out, double *s_out) {
    cplx sigma = sig_re + I * sig_im, c = c_re + I * c_im;
    const cplx *wc = (const cplx *)w, *Sc = (const cplx *)S;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
        cplx V = (wc[i] - sigma) / c;
        if (V_out) ((cplx *)V_out)[i] = V;
        if (B_out) ((cplx *)B_out)[i] = 1.0 - V;
        if (s_out) ((cplx *)s_out)[i] = Sc[i] / c;
    }
    return 0;
}

/* Plain l2 norm in a fixed sequential order (reading R-21). */
static double norm2(const cplx *a, long n) {
    double acc = 0.0;
    for (long i = 0; i < n; ++i) acc += creal(a[i]) * creal(a[i]) + cimag(a[i]) * cimag(a[i]);
    return sqrt(acc);
}

/* ---------------------------------------------------------- Algorithm 1 -- */
/*
 * form = 0 (x-form): Algorithm 1 literally:
 *     x <- 0
 *     repeat
 *        Delta <- B[(L+1)^-1 (B x + s) - x]            (line 3, "residual")
 *        x <- x + alpha Delta                           (line 4, "update")
 *     until ||Delta|| / ||Gamma^-1 s|| < eps            (line 5)
 *   with ||Gamma^-1 s|| read alpha-free as ||B (L+1)^-1 s|| (reading R-4).
 * form = 1 (Delta-form): Delta_0 = B (L+1)^-1 s and
 *     Delta_{k+1} = Delta_k + alpha B[(L+1)^-1 (B Delta_k) - Delta_k]
 *   i.e. Delta_{k+1} = (1 - Gamma^-1 A) Delta_k, same x_k.
 * Stop (reading R-5): after the update of iteration k (0-based) test
 * r_k = ||Delta_k|| / n0; return x_{k+1}, n_done = k + 1.  tol <= 0 runs
 * exactly n_max iterations.  hist[k] = r_k (if hist != NULL).
 * Returns 0 (converged or ran n_max), 1 if the residual became non-finite,
 * negative on argument errors.
 */
int orc_fixed_point(const double *w, const double *S, int ndim, const long *dims,
                    const double *h, double D, double sig_re, double sig_im, double c_re,
                    double c_im, double alpha, double tol, long n_max, int form,
                    double *x_out, double *hist, long *n_done, double *n0_out) {
    if (ndim < 1 || ndim > 3 || n_max < 1) return -2;
    long n = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        n *= dims[a];
    }
    size_t bytes = sizeof(cplx) * (size_t)n;
    cplx *B = (cplx *)malloc(bytes), *s = (cplx *)malloc(bytes);
    cplx *u = (cplx *)malloc(bytes), *Dl = (cplx *)malloc(bytes);
    cplx *x = (cplx *)x_out;
    if (!B || !s || !u || !Dl) { free(B); free(s); free(u); free(Dl); return -3; }
    orc_setup(w, S, n, sig_re, sig_im, c_re, c_im, NULL, (double *)B, (double *)s);

    /* n0 = ||B (L+1)^-1 s|| */
    memcpy(u, s, bytes);
    int rc = orc_apply_Linv((double *)u, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
    if (rc) goto done;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) Dl[i] = B[i] * u[i];
    double n0 = norm2(Dl, n);
    if (n0_out) *n0_out = n0;
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) x[i] = 0.0;
    *n_done = 0;
    if (n0 == 0.0) goto done;   /* zero source: x = 0 is exact */

    for (long k = 0; k < n_max; ++k) {
        if (form == 0) {
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) u[i] = B[i] * x[i] + s[i];
            rc = orc_apply_Linv((double *)u, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
            if (rc) goto done;
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) Dl[i] = B[i] * (u[i] - x[i]);
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) x[i] = x[i] + alpha * Dl[i];
        } else {
            /* Dl holds Delta_k here */
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) x[i] = x[i] + alpha * Dl[i];
        }
        double r = norm2(Dl, n) / n0;
        if (hist) hist[k] = r;
        *n_done = k + 1;
        if (!isfinite(r)) { rc = 1; goto done; }
        if (tol > 0.0 && r < tol) break;
        if (form == 1 && k + 1 < n_max) {
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) u[i] = B[i] * Dl[i];
            rc = orc_apply_Linv((double *)u, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
            if (rc) goto done;
#pragma omp parallel for schedule(static)
            for (long i = 0; i < n; ++i) Dl[i] = Dl[i] + alpha * B[i] * (u[i] - Dl[i]);
        }
    }
done:
    free(B); free(s); free(u); free(Dl);
    return rc;
}

/* ------------------------------------------- antisymmetrised system -- */
/*
 * Eq. 9-10: with a REAL scale c,
 *     A = c^-1 [[0, -A_raw^*], [A_raw, 0]],  L = c^-1 [[0, -L_raw^*], [L_raw, 0]],
 *     V = A - L = c^-1 [[0, -V_raw^*], [V_raw, 0]],  E = [x; x'],  s = c^-1 [-s'; S],
 * s' = 0 (no adjoint problem: x' -> 0).  A is skew-Hermitian, hence
 * accretive, for ANY A_raw, and ||V|| = max|V_raw| / c.  With v = V_raw/c
 * pointwise (V_raw = w - sigma, adjoint = conj):
 *     B = 1 - V = [[1, conj(v)], [-v, 1]]
 * and per Fourier mode, l(p) = D|p|^2 + sigma (Eq. 12's symbol), a = l/c,
 *     (L + 1)^-1 = [[1, -conj(a)], [a, 1]]^-1 = [[1, conj(a)], [-a, 1]] / (1 + |a|^2).
 * E is stored as two complex fields (x then x'); Algorithm 1 x-form
 * literally, r_k = ||Delta_k|| / ||B (L+1)^-1 s|| over both components.
 */
static int apply_Linv_anti(cplx *u1, cplx *u2, int ndim, const long *dims, const double *h, double D,
                           cplx sigma, double c) {
    int rc = orc_fftn((double *)u1, ndim, dims, 0);
    if (!rc) rc = orc_fftn((double *)u2, ndim, dims, 0);
    if (rc) return rc;
    long nx = dims[ndim - 1];
    long ny = ndim >= 2 ? dims[ndim - 2] : 1;
    long nz = ndim >= 3 ? dims[ndim - 3] : 1;
    double hx = h[ndim - 1], hy = ndim >= 2 ? h[ndim - 2] : 1.0, hz = ndim >= 3 ? h[ndim - 3] : 1.0;
#pragma omp parallel for schedule(static)
    for (long l = 0; l < nz; ++l) {
        double pz = ndim >= 3 ? freq(l, nz, hz) : 0.0;
        for (long j = 0; j < ny; ++j) {
            double py = ndim >= 2 ? freq(j, ny, hy) : 0.0;
            for (long i = 0; i < nx; ++i) {
                double px = freq(i, nx, hx);
                long q = (l * ny + j) * nx + i;
                cplx a = (D * (px * px + py * py + pz * pz) + sigma) / c;
                double det = 1.0 + creal(a) * creal(a) + cimag(a) * cimag(a);
                cplx v1 = u1[q], v2 = u2[q];
                u1[q] = (v1 + conj(a) * v2) / det;
                u2[q] = (v2 - a * v1) / det;
            }
        }
    }
    rc = orc_fftn((double *)u1, ndim, dims, 1);
    if (!rc) rc = orc_fftn((double *)u2, ndim, dims, 1);
    return rc;
}

int orc_fixed_point_anti(const double *w, const double *S, int ndim, const long *dims, const double *h,
                         double D, double sig_re, double sig_im, double c, double alpha, double tol,
                         long n_max, double *x_out, double *hist, long *n_done, double *n0_out) {
    if (ndim < 1 || ndim > 3 || n_max < 1 || !(c > 0.0)) return -2;
    long n = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        n *= dims[a];
    }
    size_t bytes = sizeof(cplx) * (size_t)n;
    cplx sigma = sig_re + I * sig_im;
    const cplx *wc = (const cplx *)w, *Sc = (const cplx *)S;
    cplx *v = malloc(bytes), *u1 = malloc(bytes), *u2 = malloc(bytes), *d1 = malloc(bytes), *d2 = malloc(bytes);
    cplx *x1 = (cplx *)x_out, *x2 = x1 + n;
    int rc = 0;
    *n_done = 0;
    if (!v || !u1 || !u2 || !d1 || !d2) { rc = -3; goto done; }
    for (long i = 0; i < n; ++i) v[i] = (wc[i] - sigma) / c;          /* V_raw / c */
    /* n0 = ||B (L+1)^-1 s||, s = [0; S/c] */
    for (long i = 0; i < n; ++i) { u1[i] = 0.0; u2[i] = Sc[i] / c; }
    rc = apply_Linv_anti(u1, u2, ndim, dims, h, D, sigma, c);
    if (rc) goto done;
    for (long i = 0; i < n; ++i) { d1[i] = u1[i] + conj(v[i]) * u2[i]; d2[i] = -v[i] * u1[i] + u2[i]; }
    double acc = 0.0;
    for (long i = 0; i < n; ++i) acc += creal(d1[i]) * creal(d1[i]) + cimag(d1[i]) * cimag(d1[i]);
    for (long i = 0; i < n; ++i) acc += creal(d2[i]) * creal(d2[i]) + cimag(d2[i]) * cimag(d2[i]);
    double n0 = sqrt(acc);
    if (n0_out) *n0_out = n0;
    for (long i = 0; i < n; ++i) { x1[i] = 0.0; x2[i] = 0.0; }
    if (n0 == 0.0) goto done;
    for (long k = 0; k < n_max; ++k) {
        /* u = B x + s */
        for (long i = 0; i < n; ++i) {
            u1[i] = x1[i] + conj(v[i]) * x2[i];
            u2[i] = -v[i] * x1[i] + x2[i] + Sc[i] / c;
        }
        rc = apply_Linv_anti(u1, u2, ndim, dims, h, D, sigma, c);
        if (rc) goto done;
        /* Delta = B (y - x); x += alpha Delta */
        acc = 0.0;
        for (long i = 0; i < n; ++i) {
            cplx e1 = u1[i] - x1[i], e2 = u2[i] - x2[i];
            cplx g1 = e1 + conj(v[i]) * e2, g2 = -v[i] * e1 + e2;
            x1[i] += alpha * g1;
            x2[i] += alpha * g2;
            acc += creal(g1) * creal(g1) + cimag(g1) * cimag(g1) + creal(g2) * creal(g2) + cimag(g2) * cimag(g2);
        }
        double r = sqrt(acc) / n0;
        if (hist) hist[k] = r;
        *n_done = k + 1;
        if (!isfinite(r)) { rc = 1; goto done; }
        if (tol > 0.0 && r < tol) break;
    }
done:
    free(v); free(u1); free(u2); free(d1); free(d2);
    return rc;
}

/* --------------------------------------------------------- BiCGSTAB -- */
/*
 * M u = B [u - (L+1)^-1 (B u)]: the preconditioned operator Gamma^-1 A of
 * Eq. 5 with alpha = 1 (a Krylov method's iterates do not
 * depend on a scalar factor of the system; reading R-25).
 */
static int apply_M(const cplx *B, const cplx *u, cplx *out, cplx *tmp, long n, int ndim, const long *dims,
                   const double *h, double D, double sig_re, double sig_im, double c_re, double c_im) {
    for (long i = 0; i < n; ++i) tmp[i] = B[i] * u[i];
    int rc = orc_apply_Linv((double *)tmp, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
    if (rc) return rc;
    for (long i = 0; i < n; ++i) out[i] = B[i] * (u[i] - tmp[i]);
    return 0;
}

/* (a, b) = sum conj(a_i) b_i in a fixed sequential order */
static cplx dotc(const cplx *a, const cplx *b, long n) {
    cplx acc = 0.0;
    for (long i = 0; i < n; ++i) acc += conj(a[i]) * b[i];
    return acc;
}

/*
 * BiCGSTAB (van der Vorst 1992; the unpreconditioned form of Saad,
 * "Iterative Methods for Sparse Linear Systems", Alg. 7.7, complex with
 * conjugated inner products) on M x = b, b = B (L+1)^-1 s (Gamma^-1 s with
 * alpha = 1), x_0 = 0, shadow residual rhat = r_0 = b:
 *     rho = (rhat, r); p = r
 *     loop j = 0, 1, ...
 *        v = M p;  a = rho / (rhat, v);  s = r - a v
 *        if ||s|| / ||b|| < tol: x += a p; stop          (half step)
 *        t = M s;  w = (t, s) / (t, t)
 *        x += a p + w s;  r = s - w t
 *        if ||r|| / ||b|| < tol: stop
 *        rho' = (rhat, r);  beta = (rho'/rho)(a/w);  p = r + beta (p - w v)
 * The residual is r = b - M x: the same quantity as Algorithm 1's Delta
 * (reading R-4), so the stopping test is comparable.  n_done counts loop
 * passes (each two applications of M); hist[2j] = ||s_j||/||b||,
 * hist[2j+1] = ||r_{j+1}||/||b|| (hist needs 2 n_max entries).  tol <= 0
 * runs exactly n_max passes.  Returns 0, 1 non-finite residual, 2 breakdown
 * (rho, (rhat, v) or (t, t) exactly 0), negative on argument errors.
 */
int orc_bicgstab(const double *w, const double *S, int ndim, const long *dims, const double *h, double D,
                 double sig_re, double sig_im, double c_re, double c_im, double tol, long n_max,
                 double *x_out, double *hist, long *n_done, double *nb_out, int *half) {
    if (ndim < 1 || ndim > 3 || n_max < 1) return -2;
    long n = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        n *= dims[a];
    }
    size_t bytes = sizeof(cplx) * (size_t)n;
    cplx *B = malloc(bytes), *sv = malloc(bytes), *r = malloc(bytes), *rh = malloc(bytes), *p = malloc(bytes);
    cplx *v = malloc(bytes), *sr = malloc(bytes), *t = malloc(bytes), *tmp = malloc(bytes);
    cplx *x = (cplx *)x_out;
    int rc = 0;
    *n_done = 0;
    *half = 0;
    if (!B || !sv || !r || !rh || !p || !v || !sr || !t || !tmp) { rc = -3; goto done; }
    orc_setup(w, S, n, sig_re, sig_im, c_re, c_im, NULL, (double *)B, (double *)sv);
    /* b = B (L+1)^-1 s; r_0 = b (x_0 = 0) */
    memcpy(tmp, sv, bytes);
    rc = orc_apply_Linv((double *)tmp, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
    if (rc) goto done;
    for (long i = 0; i < n; ++i) { r[i] = B[i] * tmp[i]; rh[i] = r[i]; p[i] = r[i]; x[i] = 0.0; }
    double nb = norm2(r, n);
    if (nb_out) *nb_out = nb;
    if (nb == 0.0) goto done;
    cplx rho = dotc(rh, r, n);
    for (long j = 0; j < n_max; ++j) {
        if (rho == 0.0) { rc = 2; goto done; }
        rc = apply_M(B, p, v, tmp, n, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
        if (rc) goto done;
        cplx rv = dotc(rh, v, n);
        if (rv == 0.0) { rc = 2; goto done; }
        cplx a = rho / rv;
        for (long i = 0; i < n; ++i) sr[i] = r[i] - a * v[i];
        double rs = norm2(sr, n) / nb;
        if (hist) hist[2 * j] = rs;
        *n_done = j + 1;
        if (!isfinite(rs)) { rc = 1; goto done; }
        if (tol > 0.0 && rs < tol) {
            for (long i = 0; i < n; ++i) x[i] += a * p[i];
            *half = 1;
            goto done;
        }
        rc = apply_M(B, sr, t, tmp, n, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
        if (rc) goto done;
        cplx tt = dotc(t, t, n);
        if (tt == 0.0) { rc = 2; goto done; }
        cplx om = dotc(t, sr, n) / tt;
        for (long i = 0; i < n; ++i) {
            x[i] += a * p[i] + om * sr[i];
            r[i] = sr[i] - om * t[i];
        }
        double rr = norm2(r, n) / nb;
        if (hist) hist[2 * j + 1] = rr;
        if (!isfinite(rr)) { rc = 1; goto done; }
        if (tol > 0.0 && rr < tol) goto done;
        cplx rho1 = dotc(rh, r, n);
        cplx beta = (rho1 / rho) * (a / om);
        for (long i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - om * v[i]);
        rho = rho1;
    }
done:
    free(B); free(sv); free(r); free(rh); free(p); free(v); free(sr); free(t); free(tmp);
    return rc;
}

/* ------------------------------------------- tensor diffusion (u, F) -- */
/*
 * PAPER.md §3.2 (L199-227), steady state (d_t = 0): F = -D grad u splits
 * div(D grad u) - mu u + S = 0 into
 *     mu u + div F = S,      D^-1 F + grad u = 0                (Eqs. 16-17)
 * i.e. A_raw [u; F] = [S; 0] with A_raw = [[mu, div], [grad, D^-1]], and
 *     L = c^-1 S^-1/2 [[mubar, div], [grad, Dbar^-1]] S^-1/2,
 *     V = c^-1 S^-1/2 [[mu - mubar, 0], [0, D^-1 - Dbar^-1]] S^-1/2,
 *     E = S^1/2 [u; F],   s = c^-1 S^-1/2 [S; 0]                 (Eq. 18)
 * with S = diag(s_u, s_F, .., s_F) (the canonical-form parameters mubar,
 * Dbar^-1, s_u, s_F, c come from oracle.py canonical_tdiff, reading R-29).
 * Per Fourier mode (grad -> i p, div -> i p^T):
 *     L + 1 = [[a, i q^T], [i q, Dm]],  a = mubar/(c s_u) + 1,
 *     q = p / (c sqrt(s_u s_F)),  Dm = Dbar^-1 / (c s_F) + I
 * inverted by its Schur complement: w = Dm^-1 q, sig = a + q^T w,
 *     out_u = (u - i w^T F) / sig
 *     out_F = Dm^-1 F - i w out_u
 * (Dm symmetric).  V per voxel: v_u = (mu - mubar)/(c s_u) and the d x d
 * block Vf = (D^-1 - Dbar^-1)/(c s_F); B = 1 - V.  Fields are stored
 * component-major: E[k][voxel], k = 0 (u), 1..d (F_x, F_y, F_z in axis
 * order x, y, z).  Algorithm 1 x-form; r_k over all components.
 *
 * Inputs: mu[n], dinv[n][d(d+1)/2] (the symmetric D^-1 per voxel, packed
 * row-major upper: 2-D xx, xy, yy; 3-D xx, xy, xz, yy, yz, zz), S[n] (real),
 * mubar, dbar[d(d+1)/2] (Dbar^-1 packed), s_u, s_F, c.  Output E[(d+1) n]
 * complex (the first component is sqrt(s_u) u).
 */
static void sym_unpack(const double *pk, int d, double M[3][3]) {
    if (d == 2) {
        M[0][0] = pk[0]; M[0][1] = M[1][0] = pk[1]; M[1][1] = pk[2];
    } else {
        M[0][0] = pk[0]; M[0][1] = M[1][0] = pk[1]; M[0][2] = M[2][0] = pk[2];
        M[1][1] = pk[3]; M[1][2] = M[2][1] = pk[4]; M[2][2] = pk[5];
    }
}

/* inverse of a symmetric d x d matrix by cofactors (d = 2, 3) */
static void sym_inv(double M[3][3], int d, double R[3][3]) {
    if (d == 2) {
        double det = M[0][0] * M[1][1] - M[0][1] * M[1][0];
        R[0][0] = M[1][1] / det; R[1][1] = M[0][0] / det;
        R[0][1] = R[1][0] = -M[0][1] / det;
        return;
    }
    double c00 = M[1][1] * M[2][2] - M[1][2] * M[2][1], c01 = M[1][2] * M[2][0] - M[1][0] * M[2][2];
    double c02 = M[1][0] * M[2][1] - M[1][1] * M[2][0];
    double det = M[0][0] * c00 + M[0][1] * c01 + M[0][2] * c02;
    R[0][0] = c00 / det; R[1][0] = c01 / det; R[2][0] = c02 / det;
    R[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) / det;
    R[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) / det;
    R[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) / det;
    R[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) / det;
    R[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) / det;
    R[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) / det;
}

static int apply_Linv_tdiff(cplx *E, long n, int ndim, const long *dims, const double *h, double a,
                            double Dm_inv[3][3], double qs) {
    int d = ndim;
    for (int k = 0; k <= d; ++k) {
        int rc = orc_fftn((double *)(E + (size_t)k * n), ndim, dims, 0);
        if (rc) return rc;
    }
    long nx = dims[ndim - 1], ny = ndim >= 2 ? dims[ndim - 2] : 1, nz = ndim >= 3 ? dims[ndim - 3] : 1;
    double hx = h[ndim - 1], hy = ndim >= 2 ? h[ndim - 2] : 1.0, hz = ndim >= 3 ? h[ndim - 3] : 1.0;
#pragma omp parallel for schedule(static)
    for (long l = 0; l < nz; ++l)
        for (long j = 0; j < ny; ++j)
            for (long i = 0; i < nx; ++i) {
                long v = (l * ny + j) * nx + i;
                double pv[3] = {freq(i, nx, hx), ndim >= 2 ? freq(j, ny, hy) : 0.0, ndim >= 3 ? freq(l, nz, hz) : 0.0};
                double q[3], w[3] = {0, 0, 0}, sig = a;
                for (int k = 0; k < d; ++k) q[k] = pv[k] * qs;
                for (int k = 0; k < d; ++k)
                    for (int m = 0; m < d; ++m) w[k] += Dm_inv[k][m] * q[m];
                for (int k = 0; k < d; ++k) sig += q[k] * w[k];
                cplx u = E[v], F[3], wF = 0.0;
                for (int k = 0; k < d; ++k) { F[k] = E[(size_t)(k + 1) * n + v]; wF += w[k] * F[k]; }
                cplx ou = (u - I * wF) / sig;
                E[v] = ou;
                for (int k = 0; k < d; ++k) {
                    cplx acc = 0.0;
                    for (int m = 0; m < d; ++m) acc += Dm_inv[k][m] * F[m];
                    E[(size_t)(k + 1) * n + v] = acc - I * w[k] * ou;
                }
            }
    for (int k = 0; k <= d; ++k) {
        int rc = orc_fftn((double *)(E + (size_t)k * n), ndim, dims, 1);
        if (rc) return rc;
    }
    return 0;
}

/* out = B in, B = 1 - V per voxel (block-diagonal) */
static void apply_B_tdiff(const cplx *in, cplx *out, long n, int d, const double *vu, const double *vf) {
    const int np = d * (d + 1) / 2;
    for (long v = 0; v < n; ++v) {
        double Vf[3][3];
        sym_unpack(vf + (size_t)v * np, d, Vf);
        out[v] = (1.0 - vu[v]) * in[v];
        for (int k = 0; k < d; ++k) {
            cplx acc = in[(size_t)(k + 1) * n + v];
            for (int m = 0; m < d; ++m) acc -= Vf[k][m] * in[(size_t)(m + 1) * n + v];
            out[(size_t)(k + 1) * n + v] = acc;
        }
    }
}

int orc_fixed_point_tdiff(const double *mu, const double *dinv, const double *S, int ndim, const long *dims,
                          const double *h, double mubar, const double *dbar, double s_u, double s_F, double c,
                          double alpha, double tol, long n_max, double *E_out, double *hist, long *n_done,
                          double *n0_out) {
    if (ndim < 2 || ndim > 3 || n_max < 1 || !(c > 0.0) || !(s_u > 0.0) || !(s_F > 0.0)) return -2;
    long n = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        n *= dims[a];
    }
    const int d = ndim, nc = d + 1, np = d * (d + 1) / 2;
    size_t bytes = sizeof(cplx) * (size_t)n * nc;
    double *vu = malloc(sizeof(double) * n), *vf = malloc(sizeof(double) * n * np);
    cplx *s = malloc(bytes), *u = malloc(bytes), *Dl = malloc(bytes), *E = (cplx *)E_out;
    int rc = 0;
    *n_done = 0;
    if (!vu || !vf || !s || !u || !Dl) { rc = -3; goto done; }
    for (long v = 0; v < n; ++v) {
        vu[v] = (mu[v] - mubar) / (c * s_u);
        for (int q = 0; q < np; ++q) vf[(size_t)v * np + q] = (dinv[(size_t)v * np + q] - dbar[q]) / (c * s_F);
    }
    double Db[3][3], Dm[3][3], Dm_inv[3][3];
    sym_unpack(dbar, d, Db);
    for (int k = 0; k < d; ++k)
        for (int m = 0; m < d; ++m) Dm[k][m] = Db[k][m] / (c * s_F) + (k == m ? 1.0 : 0.0);
    sym_inv(Dm, d, Dm_inv);
    const double a = mubar / (c * s_u) + 1.0, qs = 1.0 / (c * sqrt(s_u * s_F));
    for (size_t q = 0; q < (size_t)n * nc; ++q) s[q] = 0.0;
    for (long v = 0; v < n; ++v) s[v] = S[v] / (c * sqrt(s_u));
    /* n0 = ||B (L+1)^-1 s|| */
    memcpy(u, s, bytes);
    rc = apply_Linv_tdiff(u, n, ndim, dims, h, a, Dm_inv, qs);
    if (rc) goto done;
    apply_B_tdiff(u, Dl, n, d, vu, vf);
    double n0 = norm2(Dl, n * nc);
    if (n0_out) *n0_out = n0;
    for (size_t q = 0; q < (size_t)n * nc; ++q) E[q] = 0.0;
    if (n0 == 0.0) goto done;
    for (long k = 0; k < n_max; ++k) {
        apply_B_tdiff(E, u, n, d, vu, vf);                               /* u = B E + s */
        for (size_t q = 0; q < (size_t)n * nc; ++q) u[q] += s[q];
        rc = apply_Linv_tdiff(u, n, ndim, dims, h, a, Dm_inv, qs);
        if (rc) goto done;
        for (size_t q = 0; q < (size_t)n * nc; ++q) u[q] -= E[q];       /* Delta = B (y - E) */
        apply_B_tdiff(u, Dl, n, d, vu, vf);
        for (size_t q = 0; q < (size_t)n * nc; ++q) E[q] += alpha * Dl[q];
        double r = norm2(Dl, n * nc) / n0;
        if (hist) hist[k] = r;
        *n_done = k + 1;
        if (!isfinite(r)) { rc = 1; goto done; }
        if (tol > 0.0 && r < tol) break;
    }
done:
    free(vu); free(vf); free(s); free(u); free(Dl);
    return rc;
}

/* --------------------------------------------------------- GMRES(m) -- */
/*
 * Restarted GMRES(m) on M x = b (M, b, x_0 = 0 as orc_bicgstab; reading
 * R-28), the textbook algorithm (Saad, "Iterative Methods for Sparse Linear
 * Systems", Alg. 6.9 with Givens rotations): each cycle builds an Arnoldi
 * basis by modified Gram-Schmidt from r = b - M x, minimises ||beta e1 - H y||
 * and updates x = x + V y.  After every Arnoldi step the residual estimate
 * |g_{i+1}| / ||b|| is tested against tol (the exact residual in exact
 * arithmetic); on success x is updated with the current y and the solve
 * stops.  n_done counts Arnoldi steps (= applications of M besides the
 * restart residuals); hist[k-1] = estimate after step k (n_max entries).
 * tol <= 0 runs exactly n_max steps.  Returns 0, 1 non-finite, 2 breakdown
 * other than a lucky one, negative on argument errors.
 */
int orc_gmres(const double *w, const double *S, int ndim, const long *dims, const double *h, double D,
              double sig_re, double sig_im, double c_re, double c_im, int m, double tol, long n_max,
              double *x_out, double *hist, long *n_done, double *nb_out) {
    if (ndim < 1 || ndim > 3 || n_max < 1 || m < 1) return -2;
    long n = 1;
    for (int a = 0; a < ndim; ++a) {
        if (!is_pow2(dims[a])) return -1;
        n *= dims[a];
    }
    size_t bytes = sizeof(cplx) * (size_t)n;
    cplx *B = malloc(bytes), *sv = malloc(bytes), *b = malloc(bytes), *r = malloc(bytes), *tmp = malloc(bytes);
    cplx *V = malloc(bytes * (size_t)(m + 1));
    cplx *H = calloc((size_t)(m + 1) * m, sizeof(cplx));       /* H[i*m + j], column j */
    cplx *cs = malloc(sizeof(cplx) * m), *sn = malloc(sizeof(cplx) * m), *g = malloc(sizeof(cplx) * (m + 1));
    cplx *y = malloc(sizeof(cplx) * m);
    cplx *x = (cplx *)x_out;
    int rc = 0;
    *n_done = 0;
    if (!B || !sv || !b || !r || !tmp || !V || !H || !cs || !sn || !g || !y) { rc = -3; goto done; }
    orc_setup(w, S, n, sig_re, sig_im, c_re, c_im, NULL, (double *)B, (double *)sv);
    memcpy(tmp, sv, bytes);
    rc = orc_apply_Linv((double *)tmp, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
    if (rc) goto done;
    for (long i = 0; i < n; ++i) { b[i] = B[i] * tmp[i]; x[i] = 0.0; }
    double nb = norm2(b, n);
    if (nb_out) *nb_out = nb;
    if (nb == 0.0) goto done;
    long steps = 0;
    while (steps < n_max) {
        /* r = b - M x (x = 0 on the first cycle: r = b) */
        if (steps == 0) {
            memcpy(r, b, bytes);
        } else {
            rc = apply_M(B, x, r, tmp, n, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
            if (rc) goto done;
            for (long i = 0; i < n; ++i) r[i] = b[i] - r[i];
        }
        double beta = norm2(r, n);
        if (beta == 0.0) goto done;
        for (long i = 0; i < n; ++i) V[i] = r[i] / beta;
        for (int i = 0; i <= m; ++i) g[i] = 0.0;
        g[0] = beta;
        int k = 0, stop = 0;
        for (int j = 0; j < m && steps < n_max; ++j) {
            cplx *vj = V + (size_t)j * n, *wv = V + (size_t)(j + 1) * n;
            rc = apply_M(B, vj, wv, tmp, n, ndim, dims, h, D, sig_re, sig_im, c_re, c_im);
            if (rc) goto done;
            for (int i = 0; i <= j; ++i) {                       /* modified Gram-Schmidt */
                cplx hij = dotc(V + (size_t)i * n, wv, n);
                H[i * m + j] = hij;
                for (long q = 0; q < n; ++q) wv[q] -= hij * V[(size_t)i * n + q];
            }
            double hn = norm2(wv, n);
            H[(j + 1) * m + j] = hn;
            if (hn != 0.0)
                for (long q = 0; q < n; ++q) wv[q] /= hn;
            for (int i = 0; i < j; ++i) {                        /* previous rotations */
                cplx t = cs[i] * H[i * m + j] + sn[i] * H[(i + 1) * m + j];
                H[(i + 1) * m + j] = -conj(sn[i]) * H[i * m + j] + conj(cs[i]) * H[(i + 1) * m + j];
                H[i * m + j] = t;
            }
            /* new rotation zeroing H[j+1][j]: [c s; -conj(s) conj(c)] unitary */
            cplx hjj = H[j * m + j];
            double den = sqrt(creal(hjj) * creal(hjj) + cimag(hjj) * cimag(hjj) + hn * hn);
            if (den == 0.0) { rc = 2; goto done; }
            cs[j] = conj(hjj) / den;
            sn[j] = hn / den;
            H[j * m + j] = den;
            H[(j + 1) * m + j] = 0.0;
            g[j + 1] = -conj(sn[j]) * g[j];
            g[j] = cs[j] * g[j];
            ++steps;
            k = j + 1;
            double est = cabs(g[j + 1]) / nb;
            if (hist) hist[steps - 1] = est;
            *n_done = steps;
            if (!isfinite(est)) { rc = 1; goto done; }
            if ((tol > 0.0 && est < tol) || hn == 0.0) { stop = 1; break; }
        }
        /* y = R^-1 g (k x k upper triangular), x += V y */
        for (int i = k - 1; i >= 0; --i) {
            cplx acc = g[i];
            for (int q = i + 1; q < k; ++q) acc -= H[i * m + q] * y[q];
            y[i] = acc / H[i * m + i];
        }
        for (int i = 0; i < k; ++i)
            for (long q = 0; q < n; ++q) x[q] += y[i] * V[(size_t)i * n + q];
        if (stop) break;
    }
done:
    free(B); free(sv); free(b); free(r); free(tmp); free(V); free(H); free(cs); free(sn); free(g); free(y);
    return rc;
}

/* ---------------------------------------- smallest enclosing circle -- */

typedef struct { double x, y; } pt;

static double dist(pt a, pt b) { return hypot(a.x - b.x, a.y - b.y); }

static int inside(pt p, pt c, double r) {
    double scale = fabs(c.x) + fabs(c.y) + r + 1e-300;
    return dist(p, c) <= r + 1e-14 * scale;
}

static void circle2(pt a, pt b, pt *c, double *r) {
    c->x = 0.5 * (a.x + b.x);
    c->y = 0.5 * (a.y + b.y);
    *r = 0.5 * dist(a, b);
}

/* Circumcircle of a, b, c; collinear triples fall back to the diameter of
 * the farthest pair (the only enclosing circle through two of them). */
static void circle3(pt a, pt b, pt c, pt *o, double *r) {
    double bx = b.x - a.x, by = b.y - a.y, cx = c.x - a.x, cy = c.y - a.y;
    double d = 2.0 * (bx * cy - by * cx);
    double scale = (fabs(bx) + fabs(by)) * (fabs(cx) + fabs(cy));
    if (fabs(d) <= 1e-14 * scale || d == 0.0) {
        double dab = dist(a, b), dac = dist(a, c), dbc = dist(b, c);
        if (dab >= dac && dab >= dbc) circle2(a, b, o, r);
        else if (dac >= dbc) circle2(a, c, o, r);
        else circle2(b, c, o, r);
        return;
    }
    double b2 = bx * bx + by * by, c2 = cx * cx + cy * cy;
    double ux = (cy * b2 - by * c2) / d, uy = (bx * c2 - cx * b2) / d;
    o->x = a.x + ux;
    o->y = a.y + uy;
    *r = hypot(ux, uy);
}

/* Welzl's randomised incremental smallest-enclosing-circle (the paper cites
 * Megiddo [Megiddo83] for the same problem; the result is
 * unique).  Points are shuffled with a fixed-seed LCG so the run is
 * deterministic. */
int orc_mec(const double *re, const double *im, long n, double *cre, double *cim, double *rad) {
    if (n < 1) return -2;
    pt *p = (pt *)malloc(sizeof(pt) * (size_t)n);
    if (!p) return -3;
    for (long i = 0; i < n; ++i) { p[i].x = re[i]; p[i].y = im ? im[i] : 0.0; }
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (long i = n - 1; i > 0; --i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        long j = (long)((st >> 33) % (uint64_t)(i + 1));
        pt t = p[i]; p[i] = p[j]; p[j] = t;
    }
    pt c = p[0];
    double r = 0.0;
    for (long i = 1; i < n; ++i) {
        if (inside(p[i], c, r)) continue;
        c = p[i]; r = 0.0;
        for (long j = 0; j < i; ++j) {
            if (inside(p[j], c, r)) continue;
            circle2(p[i], p[j], &c, &r);
            for (long k = 0; k < j; ++k) {
                if (inside(p[k], c, r)) continue;
                circle3(p[i], p[j], p[k], &c, &r);
            }
        }
    }
    *cre = c.x; *cim = c.y; *rad = r;
    free(p);
    return 0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
