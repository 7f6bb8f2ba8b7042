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
#endif

/* ------------------------------------------------------------------ geometry
 * A0 (R-1..R-3): theta_a = pi*a/n_ang ("evenly distributed from 0
 * to 180 degrees"); pixel centres x_c = c-(N-1)/2, y_r = (N-1)/2-r; bin centres
 * t_j = j-(n_det-1)/2.  Ray (theta, t) = {(x,y): x cos + y sin = t}  (Eq. 1).
 * Major axis (R-3): x-major iff 4a >= n_ang and 4a <= 3 n_ang; m_a = |sin| if
 * x-major else |cos|.
 */
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
void or_project(int N, int n_det, int n_ang, int n_sel, const int *sel,
                const double *img, double *sino)
{
    double half = 0.5 * (double)(N - 1);
    for (int k = 0; k < n_sel; k++) {
        int a = sel[k];
        double th = M_PI * (double)a / (double)n_ang;
        double cs = cos(th), sn = sin(th);
        int xm = (4 * a >= n_ang && 4 * a <= 3 * n_ang);
        for (int j = 0; j < n_det; j++) {
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
void or_backproject(int N, int n_det, int n_ang, int n_sel, const int *sel,
                    const double *sino, double *img)
{
    double half = 0.5 * (double)(N - 1);
    double t0 = -0.5 * (double)(n_det - 1);
    for (size_t p = 0; p < (size_t)N * N; p++) img[p] = 0.0;
    for (int k = 0; k < n_sel; k++) {
        int a = sel[k];
        double th = M_PI * (double)a / (double)n_ang;
        double cs = cos(th), sn = sin(th);
        int xm = (4 * a >= n_ang && 4 * a <= 3 * n_ang);
        double m = xm ? fabs(sn) : fabs(cs);
        for (int r = 0; r < N; r++) {
            for (int c = 0; c < N; c++) {
                double tp = ((double)c - half) * cs + (half - (double)r) * sn;
                int j0 = (int)floor(tp - t0);
                double acc = 0.0;
                for (int j = j0 - 1; j <= j0 + 2; j++) {
                    if (j < 0 || j >= n_det) continue;
                    double tj = t0 + (double)j;
                    double w = 1.0 - fabs(tj - tp) / m;
                    if (w > 0.0) acc += (w / m) * sino[(size_t)k * n_det + j];
                }
                img[(size_t)r * N + c] += acc;
            }
        }
    }
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
void or_gd(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *d,
           const double *bprime, double c, double eta, int e1, double *u)
{
    size_t n = (size_t)N * N, l = (size_t)n_sel * n_det;
    double *s = malloc(l * sizeof(double)), *g = malloc(n * sizeof(double));
    for (int it = 0; it < e1; it++) {
        or_project(N, n_det, n_ang, n_sel, sel, u, s);
        for (size_t i = 0; i < l; i++) s[i] = s[i] - d[i];
        or_backproject(N, n_det, n_ang, n_sel, sel, s, g);
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
void or_cg(int N, int n_det, int n_ang, int n_sel, const int *sel, const double *d,
           const double *bprime, double c, int e1, double *x)
{
    size_t n = (size_t)N * N, l = (size_t)n_sel * n_det;
    double *s = malloc(l * sizeof(double));
    double *r = malloc(n * sizeof(double)), *p = malloc(n * sizeof(double));
    double *q = malloc(n * sizeof(double));
    or_project(N, n_det, n_ang, n_sel, sel, x, s);
    for (size_t i = 0; i < l; i++) s[i] = d[i] - s[i];
    or_backproject(N, n_det, n_ang, n_sel, sel, s, r);
    for (size_t i = 0; i < n; i++) { r[i] = r[i] + bprime[i] - c * x[i]; p[i] = r[i]; }
    double rr = dot(n, r, r);
    for (int it = 0; it < e1; it++) {
        or_project(N, n_det, n_ang, n_sel, sel, p, s);
        or_backproject(N, n_det, n_ang, n_sel, sel, s, q);
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
    if (P->inner == 1) or_cg(P->N, P->n_det, P->n_ang, na, sel, dm, bp, c, P->e1, x);
    else {
        double eta = P->eta1 ? P->eta1[m] : 1.0 / (2.0 * na * P->N + c);
        or_gd(P->N, P->n_det, P->n_ang, na, sel, dm, bp, c, eta, P->e1, x);
    }
}

long or_admm_run(int N, int n_det, int n_ang, int M, const int32_t *off, const int32_t *idx,
                 int n_edges, const int32_t *edges, int rule, int inner, int e1, double rho,
                 const double *eta1, int e2, double eta2, int qkind, int K, int lloyd, int quality,
                 const double *d, int iters, double *X, double *L, double *XH, int threads)
{
    or_problem P = {N, n_det, n_ang, M, off, idx, n_edges, edges, rule, inner, e1, rho, eta1,
                    e2, eta2, qkind, K, lloyd, quality};
    size_t n = (size_t)N * N;
    int *deg = calloc((size_t)M, sizeof(int)), *nb = calloc((size_t)M * M, sizeof(int));
    adjacency(&P, deg, nb);
    size_t *doff = malloc((size_t)(M + 1) * sizeof(size_t));
    doff[0] = 0;
    for (int m = 0; m < M; m++) doff[m + 1] = doff[m] + (size_t)(off[m + 1] - off[m]) * n_det;
    double *BP = malloc((size_t)M * n * sizeof(double));
    long bytes = 0;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    if (rule == 0) {
        double *S = malloc((size_t)M * n * sizeof(double));
        for (int k = 0; k < iters; k++) {
            /* b'_i from the public values of iteration k */
            for (int i = 0; i < M; i++) {
                for (size_t p = 0; p < n; p++) {
                    double s = 0.0;
                    for (int e = 0; e < deg[i]; e++) s += XH[(size_t)nb[i * M + e] * n + p];
                    BP[(size_t)i * n + p] = -L[(size_t)i * n + p] + rho * ((double)deg[i] * XH[(size_t)i * n + p] + s);
                }
            }
#pragma omp parallel for schedule(dynamic, 1)
            for (int i = 0; i < M; i++)
                local_solve(&P, i, d + doff[i], BP + (size_t)i * n, 2.0 * rho * deg[i], X + (size_t)i * n);
            bytes = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bytes)
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
        }
        free(S);
    } else {
        int32_t *roff = malloc((size_t)(M + 1) * sizeof(int32_t));
        or_partition_rows(N, M, roff);
        double *XN = malloc(n * sizeof(double));
        for (int k = 0; k < iters; k++) {
            for (int m = 0; m < M; m++)
                for (size_t p = 0; p < n; p++)
                    BP[(size_t)m * n + p] = rho * XH[p] - L[(size_t)m * n + p];
#pragma omp parallel for schedule(dynamic, 1)
            for (int m = 0; m < M; m++)
                local_solve(&P, m, d + doff[m], BP + (size_t)m * n, rho, X + (size_t)m * n);
            bytes = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bytes)
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
        }
        free(roff); free(XN);
    }
    free(deg); free(nb); free(doff); free(BP);
    return bytes;
}

/* Cost models of P:235-252: Memory(M) = D/M + 3X, Communication(M) = 2(M-1)/M X. */
double or_memory_model(int M, double D, double X) { return D / M + 3.0 * X; }
double or_comm_model(int M, double X) { return 2.0 * (M - 1) / (double)M * X; }
