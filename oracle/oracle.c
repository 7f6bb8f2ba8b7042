/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the decentralized quantized ADMM
 * tomography hot path of arXiv 2410.06106.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2410_06106_b200/).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (+ label); DESIGN.md "R-k" =
 * a reading taken where the paper is silent (listed in DESIGN.md).
 *
 * Everything is double precision, written as plain loops in the paper's order.
 * The quantizers take fp32 input and decide their integer codes in the precision
 * DESIGN.md fixes (R-16, R-18): K-means thresholds/centres fp32 with fp64 sums,
 * the DCT 8-bit map in fp64, the DCT itself in exact integers.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -fopenmp oracle.c -lm
 * (OpenMP only parallelises independent ADMM nodes for the cpu_baseline timing;
 *  results do not depend on the thread count.)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
/* threads for a loop over independent outputs: the cores the enclosing team leaves free
 * (nested inside the node-level loop of or_admm_run, all cores outside it) */
static int spare_threads(void)
{
    int t = omp_get_num_procs() / omp_get_num_threads();
    return t > 1 ? t : 1;
}
#else
static int spare_threads(void) { return 1; }
#endif

/* ------------------------------------------------------------------ geometry
 * A0 (R-1..R-3): theta_a = pi*a/n_ang ("evenly distributed from 0
 * to 180 degrees"); pixel centres x_c = c-(N-1)/2, y_r = (N-1)/2-r; bin centres
 * t_j = j-(n_det-1)/2.  Ray (theta, t) = {(x,y): x cos + y sin = t}  (Eq. 1).
 * Major axis (R-3): x-major iff 4a >= n_ang and 4a <= 3 n_ang; m_a = |sin| if
 * x-major else |cos|.
 */
/* The trig of angle a: theta_a = pi a / n_ang with the integer major-axis rule when theta is
 * NULL, else the explicit list theta[] (radians in [0, pi)) with x-major iff |sin| >= |cos|
 * (R-3 for explicit lists). */
static void joseph_trig(int a, int n_ang, const double *theta, double *cs, double *sn, int *xm)
{
    double th = theta ? theta[a] : M_PI * (double)a / (double)n_ang;
    *cs = cos(th);
    *sn = sin(th);
    if (theta) *xm = fabs(*sn) >= fabs(*cs);
    else *xm = (4 * a >= n_ang && 4 * a <= 3 * n_ang);
}

void or_angles(int n_ang, double *theta, double *cs, double *sn, int *xmajor, double *m)
{
    for (int a = 0; a < n_ang; a++) {
        double th = M_PI * (double)a / (double)n_ang;
        theta[a] = th;
        cs[a] = cos(th);
        sn[a] = sin(th);
        xmajor[a] = (4 * a >= n_ang && 4 * a <= 3 * n_ang) ? 1 : 0;
        m[a] = xmajor[a] ? fabs(sn[a]) : fabs(cs[a]);
    }
}

/* ------------------------------------------------------------------ A: forward
 * d_j = sum_i P_ji u_i  (Eq. 2) with P discretised by Joseph's method
 * (R-1): step along the ray's major axis one pixel line at a time,
 * interpolate linearly between the two pixels the ray passes between, weight 1/m_a
 * (the ray length per line).  Taps outside the grid are zero.
 * img: N*N row-major (row 0 = top).  sino: n_sel x n_det, row k = angle sel[k].
 */
void or_project_t(int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                  const double *img, double *sino)
{
    double half = 0.5 * (double)(N - 1);
    /* every (angle, bin) output is independent: OpenMP over them (when not already inside a
     * parallel region: the spare cores) changes no result */
#pragma omp parallel for collapse(2) schedule(static) num_threads(spare_threads()) if ((long)n_sel * n_det * N > (1L << 22))
    for (int k = 0; k < n_sel; k++) {
        for (int j = 0; j < n_det; j++) {
            int a = sel[k];
            double cs, sn;
            int xm;
            joseph_trig(a, n_ang, theta, &cs, &sn, &xm);
            double t = (double)j - 0.5 * (double)(n_det - 1);
            double acc = 0.0;
            if (!xm) {
                /* y-major: one sample per row r */
                for (int r = 0; r < N; r++) {
                    double y = half - (double)r;
                    double cf = (t - y * sn) / cs + half; /* fractional column */
                    double c0f = floor(cf);
                    double f = cf - c0f;
                    int c0 = (int)c0f;
                    if (c0 >= 0 && c0 < N) acc += (1.0 - f) * img[(size_t)r * N + c0];
                    if (c0 + 1 >= 0 && c0 + 1 < N) acc += f * img[(size_t)r * N + c0 + 1];
                }
                sino[(size_t)k * n_det + j] = acc / fabs(cs);
            } else {
                /* x-major: one sample per column c */
                for (int c = 0; c < N; c++) {
                    double x = (double)c - half;
                    double rf = half - (t - x * cs) / sn; /* fractional row */
                    double r0f = floor(rf);
                    double f = rf - r0f;
                    int r0 = (int)r0f;
                    if (r0 >= 0 && r0 < N) acc += (1.0 - f) * img[(size_t)r0 * N + c];
                    if (r0 + 1 >= 0 && r0 + 1 < N) acc += f * img[(size_t)(r0 + 1) * N + c];
                }
                sino[(size_t)k * n_det + j] = acc / fabs(sn);
            }
        }
    }
}

/* ------------------------------------------------------------------ A^T
 * Matched backprojector (the transpose used in Alg. 1 line 3, and Alg. 2
 * line 3).  The Joseph weight written as a closed form (R-1):
 *   P[(a,j), p] = (1/m_a) max(0, 1 - |t_j - t_p(a)| / m_a),
 *   t_p(a) = x_c cos(theta_a) + y_r sin(theta_a).
 * Pixel-driven: every bin within distance 2 of t_p is visited (all but <= 2 weights
 * are zero).
 */
void or_backproject_t(int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                      const double *sino, double *img)
{
    double half = 0.5 * (double)(N - 1);
    double t0 = -0.5 * (double)(n_det - 1);
    /* per pixel: the sum over the selected angles in their order (OpenMP over rows when not
     * already inside a parallel region; each pixel's sum is the same sequence either way) */
#pragma omp parallel for schedule(static) num_threads(spare_threads()) if ((long)n_sel * N * N > (1L << 22))
    for (int r = 0; r < N; r++) {
        for (int c = 0; c < N; c++) {
            double sum = 0.0;
            for (int k = 0; k < n_sel; k++) {
                int a = sel[k];
                double cs, sn;
                int xm;
                joseph_trig(a, n_ang, theta, &cs, &sn, &xm);
                double m = xm ? fabs(sn) : fabs(cs);
                double tp = ((double)c - half) * cs + (half - (double)r) * sn;
                int j0 = (int)floor(tp - t0);
                double acc = 0.0;
                for (int j = j0 - 1; j <= j0 + 2; j++) {
                    if (j < 0 || j >= n_det) continue;
                    double tj = t0 + (double)j;
                    double w = 1.0 - fabs(tj - tp) / m;
                    if (w > 0.0) acc += (w / m) * sino[(size_t)k * n_det + j];
                }
                sum += acc;
            }
            img[(size_t)r * N + c] = sum;
        }
    }
}

/* ------------------------------------------------------------------ Siddon
 * The paper's literal system matrix: P_ji = length of the intersection of
 * ray j with pixel i.  Siddon's algorithm (parametric ray, the sorted crossings with the
 * N+1 vertical and N+1 horizontal grid lines, one segment per pair of consecutive
 * crossings, the segment's midpoint names its pixel, its length is the weight).
 * DESIGN.md R-26: pixel (r, c) is the closed unit square x in [c - N/2, c + 1 - N/2],
 * y in [N/2 - r - 1, N/2 - r]; trig at theta = 0 and theta = pi/2 (2a = n_ang) is exact
 * (1, 0) / (0, 1); a ray lying exactly on a grid line (axis-parallel, on a pixel edge)
 * gives half of each segment's length to each of the two pixels sharing that edge (the
 * mean of the two one-sided limits; pixels outside the grid are absent).
 * Ray (theta, t): P(alpha) = t (cos, sin) + alpha (-sin, cos), unit speed.
 */
static void siddon_trig(int a, int n_ang, const double *theta, double *cs, double *sn)
{
    if (theta) { /* explicit list: exact at theta == 0 and theta == fl64(pi/2) */
        if (theta[a] == 0.0) { *cs = 1.0; *sn = 0.0; return; }
        if (theta[a] == M_PI / 2) { *cs = 0.0; *sn = 1.0; return; }
        *cs = cos(theta[a]); *sn = sin(theta[a]);
        return;
    }
    if (a == 0) { *cs = 1.0; *sn = 0.0; return; }
    if (2 * a == n_ang) { *cs = 0.0; *sn = 1.0; return; }
    double th = M_PI * (double)a / (double)n_ang;
    *cs = cos(th); *sn = sin(th);
}

static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* the (pixel, length) list of one ray; returns the count (<= 4N + 4 entries) */
static int siddon_ray(int N, double cs, double sn, double t, int *pix, double *len, double *alist)
{
    double h = 0.5 * (double)N;
    double x0 = t * cs, y0 = t * sn, dx = -sn, dy = cs;
    double amin = -INFINITY, amax = INFINITY;
    if (dx != 0.0) {
        double a1 = (-h - x0) / dx, a2 = (h - x0) / dx;
        amin = fmax(amin, fmin(a1, a2)); amax = fmin(amax, fmax(a1, a2));
    } else if (x0 < -h || x0 > h) return 0;
    if (dy != 0.0) {
        double a1 = (-h - y0) / dy, a2 = (h - y0) / dy;
        amin = fmax(amin, fmin(a1, a2)); amax = fmin(amax, fmax(a1, a2));
    } else if (y0 < -h || y0 > h) return 0;
    if (!(amax > amin)) return 0;
    int na = 0;
    alist[na++] = amin;
    alist[na++] = amax;
    for (int k = 0; k <= N; k++) {
        double g = (double)k - h; /* grid line coordinate */
        if (dx != 0.0) { double a = (g - x0) / dx; if (a > amin && a < amax) alist[na++] = a; }
        if (dy != 0.0) { double a = (g - y0) / dy; if (a > amin && a < amax) alist[na++] = a; }
    }
    qsort(alist, (size_t)na, sizeof(double), cmp_double);
    /* on a grid line: x0 (dx == 0) or y0 (dy == 0) exactly on one */
    int on_x = dx == 0.0 && floor(x0 + h) == x0 + h;
    int on_y = dy == 0.0 && floor(h - y0) == h - y0;
    int cnt = 0;
    for (int i = 0; i + 1 < na; i++) {
        double l = alist[i + 1] - alist[i];
        if (!(l > 0.0)) continue;
        double am = 0.5 * (alist[i] + alist[i + 1]);
        double xm = x0 + am * dx, ym = y0 + am * dy;
        int c = (int)floor(xm + h), r = (int)floor(h - ym);
        if (on_x) { /* columns c-1 and c share the line x = x0 */
            if (c - 1 >= 0 && c - 1 < N && r >= 0 && r < N) { pix[cnt] = r * N + c - 1; len[cnt++] = 0.5 * l; }
            if (c >= 0 && c < N && r >= 0 && r < N) { pix[cnt] = r * N + c; len[cnt++] = 0.5 * l; }
        } else if (on_y) { /* rows r-1 and r share the line y = y0 */
            if (r - 1 >= 0 && r - 1 < N && c >= 0 && c < N) { pix[cnt] = (r - 1) * N + c; len[cnt++] = 0.5 * l; }
            if (r >= 0 && r < N && c >= 0 && c < N) { pix[cnt] = r * N + c; len[cnt++] = 0.5 * l; }
        } else if (r >= 0 && r < N && c >= 0 && c < N) {
            pix[cnt] = r * N + c; len[cnt++] = l;
        }
    }
    return cnt;
}

void or_project_siddon_t(int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                         const double *img, double *sino)
{
    int *pix = malloc(sizeof(int) * (size_t)(4 * N + 8));
    double *len = malloc(sizeof(double) * (size_t)(4 * N + 8)), *al = malloc(sizeof(double) * (size_t)(2 * N + 8));
    for (int k = 0; k < n_sel; k++) {
        double cs, sn;
        siddon_trig(sel[k], n_ang, theta, &cs, &sn);
        for (int j = 0; j < n_det; j++) {
            double t = (double)j - 0.5 * (double)(n_det - 1);
            int cnt = siddon_ray(N, cs, sn, t, pix, len, al);
            double acc = 0.0;
            for (int i = 0; i < cnt; i++) acc += len[i] * img[pix[i]];
            sino[(size_t)k * n_det + j] = acc;
        }
    }
    free(pix); free(len); free(al);
}

void or_backproject_siddon_t(int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                             const double *sino, double *img)
{
    int *pix = malloc(sizeof(int) * (size_t)(4 * N + 8));
    double *len = malloc(sizeof(double) * (size_t)(4 * N + 8)), *al = malloc(sizeof(double) * (size_t)(2 * N + 8));
    for (size_t p = 0; p < (size_t)N * N; p++) img[p] = 0.0;
    for (int k = 0; k < n_sel; k++) {
        double cs, sn;
        siddon_trig(sel[k], n_ang, theta, &cs, &sn);
        for (int j = 0; j < n_det; j++) {
            double t = (double)j - 0.5 * (double)(n_det - 1);
            int cnt = siddon_ray(N, cs, sn, t, pix, len, al);
            for (int i = 0; i < cnt; i++) img[pix[i]] += len[i] * sino[(size_t)k * n_det + j];
        }
    }
    free(pix); free(len); free(al);
}

void or_project(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *img, double *sino)
{
    or_project_t(N, n_det, n_ang, NULL, n_sel, sel, img, sino);
}
void or_backproject(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *sino, double *img)
{
    or_backproject_t(N, n_det, n_ang, NULL, n_sel, sel, sino, img);
}
void or_project_siddon(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *img, double *sino)
{
    or_project_siddon_t(N, n_det, n_ang, NULL, n_sel, sel, img, sino);
}
void or_backproject_siddon(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *sino, double *img)
{
    or_backproject_siddon_t(N, n_det, n_ang, NULL, n_sel, sel, sino, img);
}

/* the projector of a run: 0 Joseph (R-1), 1 Siddon (R-26); theta NULL = uniform angles */
static void fwd(int proj, int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                const double *img, double *sino)
{
    if (proj == 1) or_project_siddon_t(N, n_det, n_ang, theta, n_sel, sel, img, sino);
    else or_project_t(N, n_det, n_ang, theta, n_sel, sel, img, sino);
}
static void bwd(int proj, int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel,
                const double *sino, double *img)
{
    if (proj == 1) or_backproject_siddon_t(N, n_det, n_ang, theta, n_sel, sel, sino, img);
    else or_backproject_t(N, n_det, n_ang, theta, n_sel, sel, sino, img);
}

/* ------------------------------------------------------------------ vectors */
static double dot(size_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (size_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------------ local solvers
 * Every local problem of the method has the form (P:158 eq:solve_u; R-7)
 *     min_x  1/2 ||A x - d||^2 + (c/2) ||x||^2 - b'^T x ,
 * i.e. (A^T A + c I) x = A^T d + b'.  paper rule: c = rho, b' = rho x^k - lambda_m;
 * graph rule: c = 2 rho deg_i, b' = -alpha_i + rho (deg_i xhat_i + S_i).
 */

/* Alg. 2: E1 gradient steps  Delta = A^T(A u - d) + c u - b', u -= eta Delta,
 * warm-started from the input u (R-9). */
void or_gd_p(int proj, int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel, const double *d,
             const double *bprime, double c, double eta, int e1, double *u)
{
    size_t n = (size_t)N * N, l = (size_t)n_sel * n_det;
    double *s = malloc(l * sizeof(double)), *g = malloc(n * sizeof(double));
    for (int it = 0; it < e1; it++) {
        fwd(proj, N, n_det, n_ang, theta, n_sel, sel, u, s);
        for (size_t i = 0; i < l; i++) s[i] = s[i] - d[i];
        bwd(proj, N, n_det, n_ang, theta, n_sel, sel, s, g);
        for (size_t i = 0; i < n; i++) {
            double delta = g[i] + c * u[i] - bprime[i];
            u[i] = u[i] - eta * delta;
        }
    }
    free(s); free(g);
}

/* Conjugate gradients on (A^T A + c I) x = A^T d + b' (config 1 "5 CG steps";
 * DESIGN.md R-8), warm start x, residual formed in sinogram space:
 *   r0 = A^T (d - A x) + b' - c x ;  p = r0
 *   repeat E1: q = A^T(A p) + c p; alpha = rr/(p.q); x += alpha p; r -= alpha q;
 *              beta = rr'/rr; p = r + beta p.
 * Guards (R-8): alpha = 0 if p.q <= 0; beta = 0 if rr == 0. */
void or_cg_p(int proj, int N, int n_det, int n_ang, const double *theta, int n_sel, const int *sel, const double *d,
             const double *bprime, double c, int e1, double *x)
{
    size_t n = (size_t)N * N, l = (size_t)n_sel * n_det;
    double *s = malloc(l * sizeof(double));
    double *r = malloc(n * sizeof(double)), *p = malloc(n * sizeof(double));
    double *q = malloc(n * sizeof(double));
    fwd(proj, N, n_det, n_ang, theta, n_sel, sel, x, s);
    for (size_t i = 0; i < l; i++) s[i] = d[i] - s[i];
    bwd(proj, N, n_det, n_ang, theta, n_sel, sel, s, r);
    for (size_t i = 0; i < n; i++) { r[i] = r[i] + bprime[i] - c * x[i]; p[i] = r[i]; }
    double rr = dot(n, r, r);
    for (int it = 0; it < e1; it++) {
        fwd(proj, N, n_det, n_ang, theta, n_sel, sel, p, s);
        bwd(proj, N, n_det, n_ang, theta, n_sel, sel, s, q);
        for (size_t i = 0; i < n; i++) q[i] = q[i] + c * p[i];
        double pq = dot(n, p, q);
        double alpha = pq > 0.0 ? rr / pq : 0.0;
        for (size_t i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        double rr2 = dot(n, r, r);
        double beta = rr > 0.0 ? rr2 / rr : 0.0;
        for (size_t i = 0; i < n; i++) p[i] = r[i] + beta * p[i];
        rr = rr2;
    }
    free(s); free(r); free(p); free(q);
}

void or_gd(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *d,
           const double *bprime, double c, double eta, int e1, double *u)
{
    or_gd_p(0, N, n_det, n_ang, NULL, n_sel, sel, d, bprime, c, eta, e1, u);
}
void or_cg(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *d,
           const double *bprime, double c, int e1, double *x)
{
    or_cg_p(0, N, n_det, n_ang, NULL, n_sel, sel, d, bprime, c, e1, x);
}

/* ------------------------------------------------------------------ K-means (Alg. 5)
 * P:277-292 "Run K-means on a ... to get the cluster centers c_1..c_k" then every
 * element -> its centre.  Made exact per DESIGN.md R-16:
 *   init   c_k = v_(floor((2k+1) n / (2K)))   (0-based order statistic, sorted fp32)
 *   Lloyd  b_k = fl32((c_k + c_{k+1}) / 2) (midpoint in fp64, one rounding);
 *          label(v) = #{k : v > b_k}  (ties -> lower cluster);
 *          c_k = fl32(sum_k / count_k) with fp64 sums; empty cluster keeps c_k;
 *   E_q Lloyd iterations, then a final assignment with the final centres.
 */
static int cmp_float(const void *a, const void *b)
{
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

static int kmeans_label(float v, const float *b, int K)
{
    int l = 0;
    for (int k = 0; k < K - 1; k++) if (v > b[k]) l++;
    return l;
}

static void kmeans_thresholds(const float *c, int K, float *b)
{
    for (int k = 0; k < K - 1; k++) b[k] = (float)(((double)c[k] + (double)c[k + 1]) * 0.5);
}

void or_kmeans_encode(const float *v, long n, int K, int iters, float *centers, int32_t *labels)
{
    float *srt = malloc((size_t)n * sizeof(float));
    memcpy(srt, v, (size_t)n * sizeof(float));
    qsort(srt, (size_t)n, sizeof(float), cmp_float);
    for (int k = 0; k < K; k++) {
        long idx = (long)(((int64_t)(2 * k + 1) * (int64_t)n) / (int64_t)(2 * K));
        centers[k] = srt[idx];
    }
    free(srt);
    float *b = malloc((size_t)(K > 1 ? K - 1 : 1) * sizeof(float));
    double *sum = malloc((size_t)K * sizeof(double));
    long *cnt = malloc((size_t)K * sizeof(long));
    for (int it = 0; it < iters; it++) {
        kmeans_thresholds(centers, K, b);
        for (int k = 0; k < K; k++) { sum[k] = 0.0; cnt[k] = 0; }
        for (long i = 0; i < n; i++) {
            int l = kmeans_label(v[i], b, K);
            sum[l] += (double)v[i];
            cnt[l] += 1;
        }
        for (int k = 0; k < K; k++)
            if (cnt[k] > 0) centers[k] = (float)(sum[k] / (double)cnt[k]);
    }
    kmeans_thresholds(centers, K, b);
    for (long i = 0; i < n; i++) labels[i] = kmeans_label(v[i], b, K);
    free(b); free(sum); free(cnt);
}

void or_kmeans_decode(const float *centers, const int32_t *labels, long n, float *out)
{
    for (long i = 0; i < n; i++) out[i] = centers[labels[i]];
}

/* ------------------------------------------------------------------ JPEG-style DCT codec
 * P:294 "each vector is encoded using the JPEG algorithm" -- read as the lossy core
 * of baseline JPEG (R-18): affine map to 8 bits with [min,max] side
 * info, level shift, 8x8 DCT, table quantisation with the standard luminance
 * table scaled to quality q, rounding; no entropy coding.  The DCT is an exact
 * integer two-pass transform with C[u][x] = round(2^14 alpha(u) cos((2x+1)u pi/16)).
 */
static const int JPEG_LUMA[64] = { /* ITU-T T.81 Annex K, Table K.1, natural order */
    16, 11, 10, 16, 24, 40, 51, 61,
    12, 12, 14, 19, 26, 58, 60, 55,
    14, 13, 16, 24, 40, 57, 69, 56,
    14, 17, 22, 29, 51, 87, 80, 62,
    18, 22, 37, 56, 68, 109, 103, 77,
    24, 35, 55, 64, 81, 104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101,
    72, 92, 95, 98, 112, 100, 103, 99};

/* IJG quality scaling: s = q<50 ? 5000/q : 200-2q; Q = clamp((Q50*s+50)/100, 1, 255). */
void or_dct_qtable(int quality, int32_t *qt)
{
    int q = quality < 1 ? 1 : (quality > 100 ? 100 : quality);
    int s = q < 50 ? 5000 / q : 200 - 2 * q;
    for (int i = 0; i < 64; i++) {
        int v = (JPEG_LUMA[i] * s + 50) / 100;
        qt[i] = v < 1 ? 1 : (v > 255 ? 255 : v);
    }
}

void or_dct_cmatrix(int32_t *C)
{
    for (int u = 0; u < 8; u++)
        for (int x = 0; x < 8; x++) {
            double al = u == 0 ? sqrt(1.0 / 8.0) : 0.5;
            C[u * 8 + x] = (int32_t)lround(16384.0 * al * cos((2.0 * x + 1.0) * u * M_PI / 16.0));
        }
}

/* floor(v / 2^k) after adding 2^(k-1): rounding right shift, floor semantics */
static int64_t rshift_round(int64_t v, int k) { return (v + ((int64_t)1 << (k - 1))) >> k; }

void or_dct_encode(const float *v, int rows, int cols, int quality, int16_t *coef, float *minmax)
{
    int32_t C[64], Q[64];
    or_dct_cmatrix(C);
    or_dct_qtable(quality, Q);
    long n = (long)rows * cols;
    float mn = v[0], mx = v[0];
    for (long i = 1; i < n; i++) { if (v[i] < mn) mn = v[i]; if (v[i] > mx) mx = v[i]; }
    minmax[0] = mn; minmax[1] = mx;
    int nbr = rows / 8, nbc = cols / 8;
    for (int br = 0; br < nbr; br++)
        for (int bc = 0; bc < nbc; bc++) {
            int16_t *out = coef + ((size_t)br * nbc + bc) * 64;
            if (mn == mx) { for (int i = 0; i < 64; i++) out[i] = 0; continue; }
            int64_t B[8][8], T[8][8];
            double den = (double)mx - (double)mn;
            for (int x = 0; x < 8; x++)
                for (int y = 0; y < 8; y++) {
                    double num = (double)v[(size_t)(8 * br + x) * cols + 8 * bc + y] - (double)mn;
                    double p = rint(num * 255.0 / den);
                    if (p < 0) p = 0;
                    if (p > 255) p = 255;
                    B[x][y] = (int64_t)p - 128;
                }
            for (int x = 0; x < 8; x++) /* rows: T = rs(B C^T, 10) */
                for (int w = 0; w < 8; w++) {
                    int64_t s = 0;
                    for (int y = 0; y < 8; y++) s += B[x][y] * C[w * 8 + y];
                    T[x][w] = rshift_round(s, 10);
                }
            for (int u = 0; u < 8; u++) /* columns: Y = C T, then quantise */
                for (int w = 0; w < 8; w++) {
                    int64_t Y = 0;
                    for (int x = 0; x < 8; x++) Y += (int64_t)C[u * 8 + x] * T[x][w];
                    int64_t D = (int64_t)Q[u * 8 + w] << 18;
                    int64_t a = Y < 0 ? -Y : Y;
                    int64_t qv = (a + D / 2) / D;
                    out[u * 8 + w] = (int16_t)(Y < 0 ? -qv : qv);
                }
        }
}

void or_dct_decode(const int16_t *coef, const float *minmax, int rows, int cols, int quality,
                   float *out, uint8_t *samples /* optional, may be NULL */)
{
    int32_t C[64], Q[64];
    or_dct_cmatrix(C);
    or_dct_qtable(quality, Q);
    float mn = minmax[0], mx = minmax[1];
    float step = (float)(((double)mx - (double)mn) / 255.0);
    int nbr = rows / 8, nbc = cols / 8;
    for (int br = 0; br < nbr; br++)
        for (int bc = 0; bc < nbc; bc++) {
            const int16_t *in = coef + ((size_t)br * nbc + bc) * 64;
            int64_t G[8][8], T[8][8];
            for (int u = 0; u < 8; u++)
                for (int w = 0; w < 8; w++) G[u][w] = (int64_t)in[u * 8 + w] * Q[u * 8 + w];
            for (int x = 0; x < 8; x++) /* T' = rs(C^T G, 10) */
                for (int w = 0; w < 8; w++) {
                    int64_t s = 0;
                    for (int u = 0; u < 8; u++) s += (int64_t)C[u * 8 + x] * G[u][w];
                    T[x][w] = rshift_round(s, 10);
                }
            for (int x = 0; x < 8; x++) /* R = T' C, sample = clamp(rs(R,18)+128) */
                for (int y = 0; y < 8; y++) {
                    int64_t R = 0;
                    for (int w = 0; w < 8; w++) R += T[x][w] * (int64_t)C[w * 8 + y];
                    int64_t smp = rshift_round(R, 18) + 128;
                    if (smp < 0) smp = 0;
                    if (smp > 255) smp = 255;
                    size_t idx = (size_t)(8 * br + x) * cols + 8 * bc + y;
                    if (samples) samples[idx] = (uint8_t)smp;
                    if (mn == mx) out[idx] = mn;
                    else {
                        volatile float prod = (float)smp * step; /* no contraction */
                        out[idx] = mn + prod;
                    }
                }
        }
}

/* ------------------------------------------------------------------ JPEG entropy coding
 * the lossless stage of "standard JPEG" after the DCT
 * quantizer -- baseline sequential Huffman coding of ITU-T T.81, written out from the
 * standard: Annex K.3 Tables K.3 / K.5 (luminance DC / AC BITS and HUFFVAL), Annex C
 * (code generation: HUFFSIZE, HUFFCODE, EHUFCO/EHUFSI), Figure A.6 (zig-zag order),
 * F.1.2.1 / F.1.2.2 (DC difference and AC run-length coding, Figures F.1-F.3, ZRL /
 * EOB), F.1.2.3 (byte stuffing: 0x00 after every 0xFF), B.2.1 / E.1.4 / F.1.2.3 (fill
 * bits are 1s; RSTm markers every R blocks with m = 0..7 cycling and the DC
 * predictor reset, F.1.4.4; R-25), F.2.2.1-F.2.2.4 (decode: DECODE with
 * MINCODE/MAXCODE/VALPTR, RECEIVE, EXTEND).  Blocks are the DCT quantizer's 8x8 blocks
 * in raster order, coefficients in natural order (row = vertical frequency) as
 * or_dct_encode writes them.  Returns the stream length, or -1 if the output capacity
 * is exceeded or a value is outside the baseline categories (DC difference > 11 bits,
 * AC > 10 bits). */
static const uint8_t JPEG_DC_BITS[16] = {0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0};
static const uint8_t JPEG_DC_VAL[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
static const uint8_t JPEG_AC_BITS[16] = {0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 0x7d};
static const uint8_t JPEG_AC_VAL[162] = {
    0x01, 0x02, 0x03, 0x00, 0x04, 0x11, 0x05, 0x12, 0x21, 0x31, 0x41, 0x06, 0x13, 0x51, 0x61, 0x07,
    0x22, 0x71, 0x14, 0x32, 0x81, 0x91, 0xa1, 0x08, 0x23, 0x42, 0xb1, 0xc1, 0x15, 0x52, 0xd1, 0xf0,
    0x24, 0x33, 0x62, 0x72, 0x82, 0x09, 0x0a, 0x16, 0x17, 0x18, 0x19, 0x1a, 0x25, 0x26, 0x27, 0x28,
    0x29, 0x2a, 0x34, 0x35, 0x36, 0x37, 0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49,
    0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59, 0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69,
    0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a, 0x83, 0x84, 0x85, 0x86, 0x87, 0x88, 0x89,
    0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a, 0xa2, 0xa3, 0xa4, 0xa5, 0xa6, 0xa7,
    0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3, 0xc4, 0xc5,
    0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe1, 0xe2,
    0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf1, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8,
    0xf9, 0xfa};

/* the tables as stored (for the pin against libjpeg's DHT segments) */
void or_jpeg_tables(uint8_t *dc_bits, uint8_t *dc_val, uint8_t *ac_bits, uint8_t *ac_val)
{
    memcpy(dc_bits, JPEG_DC_BITS, 16); memcpy(dc_val, JPEG_DC_VAL, 12);
    memcpy(ac_bits, JPEG_AC_BITS, 16); memcpy(ac_val, JPEG_AC_VAL, 162);
}

/* Annex C: HUFFSIZE (Figure C.1), HUFFCODE (Figure C.2), then EHUFCO/EHUFSI indexed by
 * symbol (Figure C.3).  Also the decoder tables of F.2.2.3 (Figure F.15): per code length
 * l = 1..16, MINCODE, MAXCODE (-1 if no codes), VALPTR. */
typedef struct {
    uint16_t ehufco[256]; uint8_t ehufsi[256];
    int32_t mincode[17], maxcode[17], valptr[17];
    const uint8_t *huffval;
} or_huff;

static void huff_build(const uint8_t *bits, const uint8_t *val, or_huff *h)
{
    int huffsize[257], huffcode[257], k = 0;
    for (int l = 1; l <= 16; l++)
        for (int i = 1; i <= bits[l - 1]; i++) huffsize[k++] = l;
    huffsize[k] = 0;
    int lastk = k, code = 0, si = huffsize[0];
    k = 0;
    while (huffsize[k]) {
        while (huffsize[k] == si) { huffcode[k] = code; code++; k++; }
        code <<= 1; si++;
    }
    memset(h->ehufsi, 0, sizeof h->ehufsi);
    for (k = 0; k < lastk; k++) { h->ehufco[val[k]] = (uint16_t)huffcode[k]; h->ehufsi[val[k]] = (uint8_t)huffsize[k]; }
    int j = 0;
    for (int l = 1; l <= 16; l++) {
        if (bits[l - 1] == 0) { h->maxcode[l] = -1; h->mincode[l] = 0; h->valptr[l] = 0; continue; }
        h->valptr[l] = j; h->mincode[l] = huffcode[j];
        j += bits[l - 1];
        h->maxcode[l] = huffcode[j - 1];
    }
    h->huffval = val;
}

/* Figure A.6: zig-zag sequence, zz[k] = natural index (row * 8 + col) of the k-th
 * coefficient, by walking the anti-diagonals, alternating direction. */
static void zigzag(int *zz)
{
    int k = 0;
    for (int s = 0; s <= 14; s++) {
        if (s % 2 == 0) { /* up-right: row decreasing */
            for (int r = (s < 8 ? s : 7); r >= 0 && s - r <= 7; r--) zz[k++] = r * 8 + (s - r);
        } else {          /* down-left: row increasing */
            for (int r = (s < 8 ? 0 : s - 7); r <= s && r <= 7; r++) zz[k++] = r * 8 + (s - r);
        }
    }
}
void or_jpeg_zigzag(int32_t *zz) { int z[64]; zigzag(z); for (int i = 0; i < 64; i++) zz[i] = z[i]; }

typedef struct { uint8_t *out; long cap, n; uint32_t acc; int nbits; int over; } or_bitw;

static void emit_byte(or_bitw *w, uint8_t b)
{
    if (w->n < w->cap) w->out[w->n] = b; else w->over = 1;
    w->n++;
}
/* append `size` bits of `code`, MSB first; 0x00 stuffed after each 0xFF data byte (F.1.2.3) */
static void put_bits(or_bitw *w, uint32_t code, int size)
{
    for (int i = size - 1; i >= 0; i--) {
        w->acc = (w->acc << 1) | ((code >> i) & 1u);
        if (++w->nbits == 8) {
            emit_byte(w, (uint8_t)w->acc);
            if ((uint8_t)w->acc == 0xFF) emit_byte(w, 0x00);
            w->acc = 0; w->nbits = 0;
        }
    }
}
static void pad_ones(or_bitw *w) { while (w->nbits) put_bits(w, 1, 1); }

static int category(int v) { int a = v < 0 ? -v : v, s = 0; while (a) { s++; a >>= 1; } return s; }

long or_jpeg_encode(const int16_t *coef, long nblocks, int restart, uint8_t *out, long cap)
{
    or_huff dc, ac;
    huff_build(JPEG_DC_BITS, JPEG_DC_VAL, &dc);
    huff_build(JPEG_AC_BITS, JPEG_AC_VAL, &ac);
    int zz[64];
    zigzag(zz);
    or_bitw w = {out, cap, 0, 0, 0, 0};
    int pred = 0;
    for (long b = 0; b < nblocks; b++) {
        if (restart > 0 && b > 0 && b % restart == 0) { /* RSTm, m = interval index mod 8 */
            pad_ones(&w);
            emit_byte(&w, 0xFF);
            emit_byte(&w, (uint8_t)(0xD0 + ((b / restart - 1) % 8)));
            pred = 0;
        }
        const int16_t *c = coef + b * 64;
        int diff = c[0] - pred; /* F.1.2.1 */
        pred = c[0];
        int s = category(diff);
        if (s > 11) return -1;
        put_bits(&w, dc.ehufco[s], dc.ehufsi[s]);
        if (s) put_bits(&w, (uint32_t)(diff < 0 ? diff - 1 : diff) & ((1u << s) - 1u), s);
        int r = 0; /* F.1.2.2, Figure F.2 */
        for (int k = 1; k < 64; k++) {
            int v = c[zz[k]];
            if (v == 0) {
                if (k == 63) put_bits(&w, ac.ehufco[0x00], ac.ehufsi[0x00]); /* EOB */
                else r++;
                continue;
            }
            while (r > 15) { put_bits(&w, ac.ehufco[0xF0], ac.ehufsi[0xF0]); r -= 16; } /* ZRL */
            int sz = category(v);
            if (sz > 10) return -1;
            int rs = (r << 4) | sz;
            put_bits(&w, ac.ehufco[rs], ac.ehufsi[rs]);
            put_bits(&w, (uint32_t)(v < 0 ? v - 1 : v) & ((1u << sz) - 1u), sz);
            r = 0;
        }
    }
    pad_ones(&w);
    return w.over ? -1 : w.n;
}

typedef struct { const uint8_t *in; long n, pos; uint32_t byte; int cnt; int marker; } or_bitr;

/* NEXTBIT (Figure F.18): a 0xFF data byte is followed by a stuffed 0x00; a marker
 * (0xFF, non-zero) stops the bit supply -- the decoder then reads zeros and flags it. */
static int next_bit(or_bitr *r)
{
    if (r->cnt == 0) {
        if (r->pos >= r->n || r->marker) { r->marker = 1; r->byte = 0; r->cnt = 8; }
        else {
            r->byte = r->in[r->pos++];
            if (r->byte == 0xFF) {
                if (r->pos < r->n && r->in[r->pos] == 0x00) r->pos++;
                else { r->pos--; r->marker = 1; r->byte = 0; }
            }
            r->cnt = 8;
        }
    }
    r->cnt--;
    return (r->byte >> r->cnt) & 1;
}
static int decode_sym(or_bitr *r, const or_huff *h) /* DECODE, Figure F.16 */
{
    int code = next_bit(r), l = 1;
    while (code > h->maxcode[l]) {
        if (++l > 16) return -1;
        code = (code << 1) | next_bit(r);
    }
    return h->huffval[h->valptr[l] + code - h->mincode[l]];
}
static int receive_extend(or_bitr *r, int s) /* RECEIVE (F.17) and EXTEND (F.12) */
{
    int v = 0;
    for (int i = 0; i < s; i++) v = (v << 1) | next_bit(r);
    if (s && v < (1 << (s - 1))) v = v - (1 << s) + 1;
    return v;
}

/* returns 0, or -1 for a malformed stream (bad code, missing / wrong RSTm, bits left over) */
int or_jpeg_decode(const uint8_t *in, long nbytes, long nblocks, int restart, int16_t *coef)
{
    or_huff dc, ac;
    huff_build(JPEG_DC_BITS, JPEG_DC_VAL, &dc);
    huff_build(JPEG_AC_BITS, JPEG_AC_VAL, &ac);
    int zz[64];
    zigzag(zz);
    or_bitr r = {in, nbytes, 0, 0, 0, 0};
    int pred = 0;
    for (long b = 0; b < nblocks; b++) {
        if (restart > 0 && b > 0 && b % restart == 0) {
            r.cnt = 0; /* discard the fill bits of the current byte */
            if (r.pos + 1 >= r.n || in[r.pos] != 0xFF || in[r.pos + 1] != 0xD0 + ((b / restart - 1) % 8)) return -1;
            r.pos += 2; r.marker = 0; pred = 0;
        }
        int16_t *c = coef + b * 64;
        for (int i = 0; i < 64; i++) c[i] = 0;
        int s = decode_sym(&r, &dc);
        if (s < 0 || s > 11) return -1;
        pred += receive_extend(&r, s);
        c[0] = (int16_t)pred;
        for (int k = 1; k < 64; k++) { /* Figure F.13 */
            int rs = decode_sym(&r, &ac);
            if (rs < 0) return -1;
            int run = rs >> 4, sz = rs & 15;
            if (sz == 0) {
                if (run == 15) { k += 15; continue; } /* ZRL */
                break;                                 /* EOB */
            }
            k += run;
            if (k > 63) return -1;
            c[zz[k]] = (int16_t)receive_extend(&r, sz);
        }
        if (r.marker && r.pos >= r.n) return -1; /* ran past the data */
    }
    /* everything consumed: the remaining bits of the last byte are fill 1s */
    if (r.cnt && ((r.byte & ((1u << r.cnt) - 1u)) != ((1u << r.cnt) - 1u))) return -1;
    return r.pos == nbytes ? 0 : -1;
}

/* ------------------------------------------------------------------ partitions
 * Angle partition: round-robin -- node m holds angles a = m (mod M);
 * contiguous (config 1) -- consecutive blocks, the first n_ang mod M nodes one
 * larger (R-5).  Writes offsets[M+1] and idx[n_ang]. */
void or_partition_angles(int n_ang, int M, int contiguous, int32_t *offsets, int32_t *idx)
{
    int pos = 0;
    offsets[0] = 0;
    for (int m = 0; m < M; m++) {
        if (contiguous) {
            int base = n_ang / M, rem = n_ang % M;
            int start = m * base + (m < rem ? m : rem);
            int cnt = base + (m < rem ? 1 : 0);
            for (int k = 0; k < cnt; k++) idx[pos++] = start + k;
        } else {
            for (int a = m; a < n_ang; a += M) idx[pos++] = a;
        }
        offsets[m + 1] = pos;
    }
}

/* Segment partition of x ("partition the variable x into M segments";
 * DESIGN.md R-6): contiguous row blocks, heights differing by at most one, the
 * first N mod M segments one row taller.  Writes row_off[M+1]. */
void or_partition_rows(int N, int M, int32_t *row_off)
{
    int base = N / M, rem = N % M;
    row_off[0] = 0;
    for (int m = 0; m < M; m++) row_off[m + 1] = row_off[m] + base + (m < rem ? 1 : 0);
}

/* ------------------------------------------------------------------ quantizer Q
 * Q applied to an exchanged vector (P:268 eq-compact:conc3).  Input rounded to
 * fp32 (the wire format); output fp32 promoted back to fp64.
 * kind: 0 none (identity, no rounding), 1 K-means, 2 DCT.
 * bytes: payload size in bytes (R-17). */
static long quantize(int kind, int K, int iters, int quality, const double *x, int rows, int cols,
                     double *xh, int32_t *labels_out)
{
    long n = (long)rows * cols;
    if (kind == 0) {
        for (long i = 0; i < n; i++) xh[i] = x[i];
        return 4 * n;
    }
    float *v = malloc((size_t)n * sizeof(float)), *o = malloc((size_t)n * sizeof(float));
    for (long i = 0; i < n; i++) v[i] = (float)x[i];
    long bytes;
    if (kind == 1) {
        float *cen = malloc((size_t)K * sizeof(float));
        int32_t *lab = labels_out ? labels_out : malloc((size_t)n * sizeof(int32_t));
        or_kmeans_encode(v, n, K, iters, cen, lab);
        or_kmeans_decode(cen, lab, n, o);
        int bits = 0;
        while ((1 << bits) < K) bits++;
        bytes = 4L * K + 4L * bits * ((n + 31) / 32);
        if (!labels_out) free(lab);
        free(cen);
    } else {
        int16_t *cf = malloc((size_t)n * sizeof(int16_t));
        float mm[2];
        or_dct_encode(v, rows, cols, quality, cf, mm);
        or_dct_decode(cf, mm, rows, cols, quality, o, NULL);
        bytes = 2 * n + 8;
        free(cf);
    }
    for (long i = 0; i < n; i++) xh[i] = (double)o[i];
    free(v); free(o);
    return bytes;
}

/* ------------------------------------------------------------------ the ADMM outer loop
 * One problem = one slice: M nodes, node m owns angles idx[off[m]..off[m+1]) and
 * the matching sinogram rows d (node-major, concatenated).
 *
 * rule 1 "paper" (P:158-166 eq:solve_u/eq:solve_x/eq:conc/eq:solve_lamda, Alg. 4 P:207-229,
 *   with Q per P:268):  state X = u_m, L = lambda_m, XG = consensus x (n values).
 *   u_m   <- inner solve of eq:solve_u (c = rho, b' = rho x - lambda_m), warm start
 *   x[m]  <- Alg. 3: E2 steps of x[m] -= eta2 rho (x[m] - u_m - lambda_m/rho),
 *            started from the current x[m]
 *   x     <- conc(Q(x[1]), ..., Q(x[M]))
 *   lambda_m <- lambda_m + rho (u_m - x)
 * rule 2 "consensus" (the standard consensus ADMM of P:121-131, eq-compact:solve_u /
 *   eq-compact:solve_x / eq-compact:solve_lambda, with x sharded in the paper's segments
 *   and Q applied to each segment as in P:268):  state X = u_m, L = lambda_m,
 *   XG = x.  u_m <- inner solve with c = rho, b' = rho x - lambda_m (as rule 1);
 *   x[m] <- (1/M) sum_n (u_n + lambda_n/rho)[m]  (the argmin of eq-compact:solve_x);
 *   x <- conc(Q(x[1]), ..., Q(x[M]));  lambda_m <- lambda_m + rho (u_m - x).
 * rule 0 "graph" (decentralized consensus ADMM over the graph, R-7):
 *   state X = x_i (private), L = alpha_i, XH = xhat_i = Q(x_i) (public).
 *   b'_i = -alpha_i + rho (deg_i xhat_i + S_i), c_i = 2 rho deg_i, S_i = sum_{j in N(i)} xhat_j
 *   x_i  <- inner solve (warm start)
 *   xhat_i <- Q(x_i);  S_i <- sum_{j in N(i)} xhat_j
 *   alpha_i <- alpha_i + rho (deg_i xhat_i - S_i)
 * inner: 0 GD (Alg. 2) with eta1[m] (if eta1 == NULL: 1/(2 a_m N + c_m), R-8), 1 CG.
 * Returns payload bytes sent per iteration summed over nodes (graph: deg*payload;
 * paper: (M-1)*segment payload).
 */
typedef struct {
    int N, n_det, n_ang, M;
    const int32_t *off, *idx;       /* angle partition */
    int n_edges; const int32_t *edges; /* 2*n_edges */
    int rule, inner, e1;
    double rho; const double *eta1;
    int e2; double eta2;
    int qkind, K, lloyd, quality;
    int proj;                        /* 0 Joseph (R-1), 1 Siddon (R-26) */
    const double *theta;             /* explicit angles (radians) or NULL: pi a / n_ang */
} or_problem;

/* Alg. 3 for one element of the owned segment x[m]:
 * repeat E2: Delta = rho (x - u - lambda/rho); x = x - eta2 Delta. */
double or_alg3(double x, double u, double lam, double rho, double eta2, int e2)
{
    for (int it = 0; it < e2; it++) {
        double delta = rho * (x - u - lam / rho);
        x = x - eta2 * delta;
    }
    return x;
}

static void adjacency(const or_problem *P, int *deg, int *nb /* M*M */)
{
    for (int i = 0; i < P->M; i++) deg[i] = 0;
    for (int e = 0; e < P->n_edges; e++) {
        int i = P->edges[2 * e], j = P->edges[2 * e + 1];
        nb[i * P->M + deg[i]++] = j;
        nb[j * P->M + deg[j]++] = i;
    }
}

static void local_solve(const or_problem *P, int m, const double *dm, const double *bp, double c,
                        double *x)
{
    int na = P->off[m + 1] - P->off[m];
    const int *sel = P->idx + P->off[m];
    if (P->inner == 1) or_cg_p(P->proj, P->N, P->n_det, P->n_ang, P->theta, na, sel, dm, bp, c, P->e1, x);
    else {
        double eta = P->eta1 ? P->eta1[m] : 1.0 / (2.0 * na * P->N + c);
        or_gd_p(P->proj, P->N, P->n_det, P->n_ang, P->theta, na, sel, dm, bp, c, eta, P->e1, x);
    }
}

/* The stopping test of P:330 ("stopping criterion of 1e-6"; R-13): the relative
 * change ||x^{k+1} - x^k|| / ||x^{k+1}|| of the iterate (0/0 := 0), maximised over the
 * iterates compared (graph rule: every node's private x_i; paper / consensus: x). */
static double rel_change(const double *cur, const double *prev, size_t n)
{
    double dd = 0.0, xx = 0.0;
    for (size_t p = 0; p < n; p++) {
        double e = cur[p] - prev[p];
        dd += e * e;
        xx += cur[p] * cur[p];
    }
    if (dd == 0.0) return 0.0;
    return xx > 0.0 ? sqrt(dd / xx) : INFINITY;
}

/* stop_tol > 0: stop after the first iteration whose relative change is <= stop_tol;
 * *iters_done (if not NULL) = iterations performed; *last_change = the last test value. */
long or_admm_run(int N, int n_det, int n_ang, int M, const int32_t *off, const int32_t *idx,
                 int n_edges, const int32_t *edges, int rule, int inner, int e1, double rho,
                 const double *eta1, int e2, double eta2, int qkind, int K, int lloyd, int quality,
                 const double *d, int iters, double *X, double *L, double *XH, int threads, int proj,
                 const double *theta, double stop_tol, int *iters_done, double *last_change)
{
    or_problem P = {N, n_det, n_ang, M, off, idx, n_edges, edges, rule, inner, e1, rho, eta1,
                    e2, eta2, qkind, K, lloyd, quality, proj, theta};
    int done = 0;
    double change = -1.0;
    size_t n = (size_t)N * N;
    int *deg = calloc((size_t)M, sizeof(int)), *nb = calloc((size_t)M * M, sizeof(int));
    adjacency(&P, deg, nb);
    size_t *doff = malloc((size_t)(M + 1) * sizeof(size_t));
    doff[0] = 0;
    for (int m = 0; m < M; m++) doff[m + 1] = doff[m] + (size_t)(off[m + 1] - off[m]) * n_det;
    double *BP = malloc((size_t)M * n * sizeof(double));
    long bytes = 0;
    /* node-level threads; with one node thread the projector loops use every core (nesting
     * under several node threads measured slower than node-level threads alone) */
    int nt = threads > 0 ? threads : 1;
#ifdef _OPENMP
    omp_set_max_active_levels(nt > 1 ? 1 : 2);
#endif
#ifndef _OPENMP
    (void)nt;
#endif
    if (rule == 0) {
        double *S = malloc((size_t)M * n * sizeof(double));
        double *XP = stop_tol > 0.0 ? malloc((size_t)M * n * sizeof(double)) : NULL;
        for (int k = 0; k < iters; k++) {
            if (XP) memcpy(XP, X, (size_t)M * n * sizeof(double));
            /* b'_i from the public values of iteration k */
            for (int i = 0; i < M; i++) {
                for (size_t p = 0; p < n; p++) {
                    double s = 0.0;
                    for (int e = 0; e < deg[i]; e++) s += XH[(size_t)nb[i * M + e] * n + p];
                    BP[(size_t)i * n + p] = -L[(size_t)i * n + p] + rho * ((double)deg[i] * XH[(size_t)i * n + p] + s);
                }
            }
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
            for (int i = 0; i < M; i++)
                local_solve(&P, i, d + doff[i], BP + (size_t)i * n, 2.0 * rho * deg[i], X + (size_t)i * n);
            bytes = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bytes) num_threads(nt)
            for (int i = 0; i < M; i++) {
                long b = quantize(qkind, K, lloyd, quality, X + (size_t)i * n, N, N, XH + (size_t)i * n, NULL);
                bytes += b * deg[i];
            }
            for (int i = 0; i < M; i++)
                for (size_t p = 0; p < n; p++) {
                    double s = 0.0;
                    for (int e = 0; e < deg[i]; e++) s += XH[(size_t)nb[i * M + e] * n + p];
                    S[(size_t)i * n + p] = s;
                }
            for (int i = 0; i < M; i++)
                for (size_t p = 0; p < n; p++)
                    L[(size_t)i * n + p] += rho * ((double)deg[i] * XH[(size_t)i * n + p] - S[(size_t)i * n + p]);
            done = k + 1;
            if (XP) {
                change = 0.0;
                for (int i = 0; i < M; i++)
                    change = fmax(change, rel_change(X + (size_t)i * n, XP + (size_t)i * n, n));
                if (change <= stop_tol) break;
            }
        }
        free(S);
        free(XP);
    } else {
        int32_t *roff = malloc((size_t)(M + 1) * sizeof(int32_t));
        or_partition_rows(N, M, roff);
        double *XN = malloc(n * sizeof(double));
        double *XP = stop_tol > 0.0 ? malloc(n * sizeof(double)) : NULL;
        for (int k = 0; k < iters; k++) {
            if (XP) memcpy(XP, XH, n * sizeof(double));
            for (int m = 0; m < M; m++)
                for (size_t p = 0; p < n; p++)
                    BP[(size_t)m * n + p] = rho * XH[p] - L[(size_t)m * n + p];
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
            for (int m = 0; m < M; m++)
                local_solve(&P, m, d + doff[m], BP + (size_t)m * n, rho, X + (size_t)m * n);
            bytes = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bytes) num_threads(nt)
            for (int m = 0; m < M; m++) {
                size_t lo = (size_t)roff[m] * N, hi = (size_t)roff[m + 1] * N;
                double *seg = malloc((hi - lo) * sizeof(double));
                for (size_t p = lo; p < hi; p++) {
                    if (rule == 1) {
                        seg[p - lo] = or_alg3(XH[p], X[(size_t)m * n + p], L[(size_t)m * n + p], rho, eta2, e2);
                    } else {  /* consensus: the mean over all nodes, summed in node order */
                        double acc = 0.0;
                        for (int q = 0; q < M; q++) acc += X[(size_t)q * n + p] + L[(size_t)q * n + p] / rho;
                        seg[p - lo] = acc / (double)M;
                    }
                }
                long b = quantize(qkind, K, lloyd, quality, seg, roff[m + 1] - roff[m], N, XN + lo, NULL);
                bytes += b * (M - 1);
                free(seg);
            }
            memcpy(XH, XN, n * sizeof(double));
            for (int m = 0; m < M; m++)
                for (size_t p = 0; p < n; p++)
                    L[(size_t)m * n + p] += rho * (X[(size_t)m * n + p] - XH[p]);
            done = k + 1;
            if (XP) {
                change = rel_change(XH, XP, n);
                if (change <= stop_tol) break;
            }
        }
        free(roff); free(XN); free(XP);
    }
    if (iters_done) *iters_done = done;
    if (last_change) *last_change = change;
    free(deg); free(nb); free(doff); free(BP);
    return bytes;
}

/* Cost models of P:235-252: Memory(M) = D/M + 3X, Communication(M) = 2(M-1)/M X. */
double or_memory_model(int M, double D, double X) { return D / M + 3.0 * X; }
double or_comm_model(int M, double X) { return 2.0 * (M - 1) / (double)M * X; }
