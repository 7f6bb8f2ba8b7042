// solver.cu -- see solver.cuh.
#include <math.h>

#include "solver.cuh"

namespace tq {

void DevGeom::init(int N_, int n_ang_, int n_det_, int proj_, const double *angles_rad) {
    projector_setup();
    N = N_; n_ang = n_ang_; n_det = n_det_; proj = proj_;
    n = (long long)N * N;
    std::vector<AngleHost> a = make_angles(n_ang, angles_rad);
    std::vector<double2> t(n_ang);
    std::vector<int> xm(n_ang);
    for (int i = 0; i < n_ang; i++) {
        t[i] = make_double2(a[i].cs, a[i].sn);
        // R-26: exact trig at pi/2 (uniform angles: 2a = n_ang; explicit: theta == fl64(pi/2))
        const bool half_pi = angles_rad ? angles_rad[i] == M_PI / 2 : 2 * i == n_ang;
        if (proj == 1 && half_pi) t[i] = make_double2(0.0, 1.0);
        xm[i] = a[i].xmajor;
    }
    TQ_CHECK_CUDA(cudaMalloc(&trig, sizeof(double2) * n_ang));
    TQ_CHECK_CUDA(cudaMalloc(&xmaj, sizeof(int) * n_ang));
    TQ_CHECK_CUDA(cudaMemcpy(trig, t.data(), sizeof(double2) * n_ang, cudaMemcpyHostToDevice));
    TQ_CHECK_CUDA(cudaMemcpy(xmaj, xm.data(), sizeof(int) * n_ang, cudaMemcpyHostToDevice));
    xmaj_h = xm;
}

void DevGeom::release() {
    if (trig) cudaFree(trig);
    if (xmaj) cudaFree(xmaj);
    trig = nullptr; xmaj = nullptr;
}

void Inner::init(int prec_, const DevGeom &g, const std::vector<std::vector<int>> &angles) {
    prec = prec_;
    L = (int)angles.size();
    n = g.n;
    rows_h.clear(); row0_h.clear(); nang_h.clear();
    for (int i = 0; i < L; i++) {
        row0_h.push_back((int)rows_h.size());
        nang_h.push_back((int)angles[i].size());
        for (size_t k = 0; k < angles[i].size(); k++) rows_h.push_back(RayRow{i, angles[i][k], (int)k, 0});
    }
    n_rows = (int)rows_h.size();
    std::vector<int> ol, of(1, 0);
    for (int i = 0; i < L; i++)
        for (int o = 0; o < 2; o++) {
            for (int r = row0_h[i]; r < row0_h[i] + nang_h[i]; r++)
                if (g.xmaj_h[rows_h[r].angle] == o) ol.push_back(r);
            of.push_back((int)ol.size());
        }
    nt_line = ceil_div(g.N, FP_TH);
    nt_cross = ceil_div(g.N, FP_TW);
    sp = g.n_det + 2;
    int max_nang = 0;
    for (int c : nang_h) max_nang = std::max(max_nang, c);
    // partials per node: backprojector tiles, vector blocks, or the forward reduction's CTAs
    // (angles x bin blocks of >= 32 bins) of a CG step
    part_stride = std::max({bp_tiles(g.N), vec_blocks(n), max_nang * ceil_div(g.n_det, 32), 1});
    const size_t es = esize();
    auto A = [&](void **p, size_t bytes) {
        TQ_CHECK_CUDA(cudaMalloc(p, std::max<size_t>(bytes, 16)));
        TQ_CHECK_CUDA(cudaMemset(*p, 0, std::max<size_t>(bytes, 16)));
    };
    A((void **)&rows, sizeof(RayRow) * n_rows);
    A((void **)&row0, sizeof(int) * L);
    A((void **)&nang, sizeof(int) * L);
    TQ_CHECK_CUDA(cudaMemcpy(rows, rows_h.data(), sizeof(RayRow) * n_rows, cudaMemcpyHostToDevice));
    TQ_CHECK_CUDA(cudaMemcpy(row0, row0_h.data(), sizeof(int) * L, cudaMemcpyHostToDevice));
    TQ_CHECK_CUDA(cudaMemcpy(nang, nang_h.data(), sizeof(int) * L, cudaMemcpyHostToDevice));
    A((void **)&olist, sizeof(int) * ol.size());
    A((void **)&oofs, sizeof(int) * of.size());
    if (!ol.empty()) TQ_CHECK_CUDA(cudaMemcpy(olist, ol.data(), sizeof(int) * ol.size(), cudaMemcpyHostToDevice));
    TQ_CHECK_CUDA(cudaMemcpy(oofs, of.data(), sizeof(int) * of.size(), cudaMemcpyHostToDevice));
    const size_t nwin = (size_t)n_rows * nt_line * nt_cross;
    A(&fpart, es * (size_t)n_rows * nt_line * 2 * fp_ps(g.n_det));
    A((void **)&fwin, sizeof(FpWin) * nwin);
    A((void **)&frg, sizeof(FpRowGeo) * n_rows);
    n_olist = (int)ol.size();
    A((void **)&frec, sizeof(FpRec) * (size_t)nt_line * nt_cross * std::max(1, n_olist));
    A((void **)&futab, sizeof(FpUnitTab) * 2 * (size_t)std::max(1, L) * nt_line * nt_cross);
    launch_fp_setup(rows, g.xmaj, g.trig, n_rows, g.N, g.n_det, fwin, frg, olist, n_olist, frec, oofs, L, futab, 0);
    A((void **)&rowc, sizeof(double4) * std::max(1, n_rows));
    launch_bp_rowc(rows, g.trig, g.xmaj, n_rows, rowc, 0);
    TQ_CHECK_CUDA(cudaDeviceSynchronize());
    for (void **v : {&X, &R, &P, &Q, &BP}) A(v, es * n * L);
    A(&D, es * (size_t)n_rows * g.n_det);
    A(&AX, es * (size_t)n_rows * g.n_det);
    // S rows carry a zero guard bin at 0 and n_det + 1; SPAD zero elements before and after the
    // whole array let the backprojector stage its fixed 96-bin windows without bounds checks
    A(&S_base, es * ((size_t)n_rows * sp + 2 * SPAD));
    S = (uint8_t *)S_base + es * SPAD;
    A((void **)&cnode, sizeof(double) * L);
    A((void **)&eta, sizeof(double) * L);
    A((void **)&scal, sizeof(double) * S_NSLOT * L);
    A((void **)&partial, sizeof(double) * (size_t)part_stride * L);
    A((void **)&cgs, sizeof(double) * (size_t)part_stride * L);
    A((void **)&cgp, sizeof(double) * (size_t)part_stride * L);
    A((void **)&counter, sizeof(unsigned) * L);
}

void Inner::release() {
    for (void *p : {(void *)rows, (void *)row0, (void *)nang, X, R, P, Q, BP, D, AX, S_base, (void *)cnode,
                    (void *)eta, (void *)scal, (void *)partial, (void *)cgs, (void *)cgp, (void *)counter, (void *)rowc, (void *)olist,
                    (void *)oofs, fpart, (void *)fwin, (void *)frg, (void *)frec, (void *)futab})
        if (p) cudaFree(p);
    rows = nullptr; row0 = nang = olist = oofs = nullptr;
    fpart = nullptr; fwin = nullptr; frg = nullptr; frec = nullptr; futab = nullptr;
    X = R = P = Q = BP = D = AX = S = S_base = nullptr;
    cnode = eta = scal = partial = cgs = cgp = nullptr;
    counter = nullptr;
    rowc = nullptr;
}

int Inner::project(const DevGeom &g, const void *img, bool resid, cudaStream_t st, void *out,
                   int out_stride, int out_off, bool cg, int n0, int cnt) {
    if (!out) { out = S; out_stride = sp; out_off = 1; }
    if (cnt < 0) cnt = L - n0;
    const bool grp = n0 != 0 || cnt != L;
    // a node group [n0, n0 + cnt): its images, unit groups and (contiguous) ray rows
    const int rb = n0 < L ? row0_h[n0] : n_rows, nr = (n0 + cnt < L ? row0_h[n0 + cnt] : n_rows) - rb;
    if (prec == 0) {
        TQ_REQUIRE(!grp || (g.N % 4 == 0 && frec), "node groups need the persistent fp32 forward kernel");
        FpArgs<float> a{(const float *)img + n * n0, n, g.N, g.n_det, olist, oofs + 2 * n0, fwin, frg, (float *)fpart,
                        nt_line, nt_cross, kMagicBits4, frec, n_olist, cnt, futab, g.proj, n0, L};
        launch_fp(0, &a, cnt, st);
        FpRedArgs<float> r{(const float *)fpart, rows, g.trig, g.xmaj, (const float *)D, (float *)out,
                           out_stride, out_off, g.N, g.n_det, nt_line, rowc, frg, nt_cross,
                           cg ? 1 : 0, cgs, part_stride, rb};
        launch_fp_reduce(0, resid, &r, nr, g.n_det, st);
    } else {
        TQ_REQUIRE(!grp, "node groups are fp32 only");
        FpArgs<double> a{(const double *)img, n, g.N, g.n_det, olist, oofs, fwin, frg, (double *)fpart,
                         nt_line, nt_cross, kMagicBits4, frec, n_olist, L, futab, g.proj, 0, L};
        launch_fp(1, &a, L, st);
        FpRedArgs<double> r{(const double *)fpart, rows, g.trig, g.xmaj, (const double *)D,
                            (double *)out, out_stride, out_off, g.N, g.n_det, nt_line, rowc, nullptr, nt_cross,
                            cg ? 1 : 0, cgs, part_stride, 0};
        launch_fp_reduce(1, resid, &r, n_rows, g.n_det, st);
    }
    return 3;
}

int Inner::backproject(const DevGeom &g, int epi, void *out, void *out2, const void *vin, cudaStream_t st,
                       const void *rin, int n0, int cnt) {
    const void *b2 = epi == EPI_CGR ? rin : BP;  // second epilogue operand: b' (RESID, GD) or r (CGR)
    if (cnt < 0) cnt = L - n0;
    // a node group: every node-indexed table and node-major vector starts at node n0 (the
    // sinogram rows are addressed through the absolute node_row0 values)
    const long long o = n * n0;
    if (prec == 0) {
        auto f = [o](const void *p) { return p ? (float *)p + o : nullptr; };
        BpArgs<float> a{(const float *)S, sp, 1, row0 + n0, nang + n0, rows, g.trig, g.xmaj, g.N, g.n_det, n,
                        f(out), f(out2), f(vin), f(b2), cnode + n0, eta + n0,
                        partial + (long long)part_stride * n0, counter + n0, scal + (long long)S_NSLOT * n0,
                        part_stride, kMagicBits4, g.proj, rowc};
        launch_bp(0, epi, &a, cnt, g.N, st);
    } else {
        auto f = [o](const void *p) { return p ? (double *)p + o : nullptr; };
        BpArgs<double> a{(const double *)S, sp, 1, row0 + n0, nang + n0, rows, g.trig, g.xmaj, g.N, g.n_det, n,
                         f(out), f(out2), f(vin), f(b2), cnode + n0, eta + n0,
                         partial + (long long)part_stride * n0, counter + n0, scal + (long long)S_NSLOT * n0,
                         part_stride, kMagicBits4, g.proj, rowc};
        launch_bp(1, epi, &a, cnt, g.N, st);
    }
    return 1;
}

// CG on (A^T A + c I) x = A^T d + b' from the warm start X (R-8):
// r0 = A^T(d - A x) + b' - c x (sinogram-space residual), p0 = r0, then E1 steps of
//   s = A p;  alpha = rr / p.q with p.q = ||s||^2 + c ||p||^2   (forward reduction)
//   r -= alpha (A^T s + c p);  beta = rr_new / rr              (backprojector epilogue)
//   x += alpha p;  p = r + beta p;  ||p||^2                     (vector pass)
// -- p.q = p.(A^T A p + c p) written through A p, so q is never stored and the residual
// update rides on the backprojection; the last step needs neither r nor beta (the next
// solve restarts from the residual backprojection), so it has no backprojection at all.
int Inner::cg(const DevGeom &g, int e1, cudaStream_t st, int ax, int n0, int cnt) {
    if (cnt < 0) cnt = L - n0;
    const int rb = n0 < L ? row0_h[n0] : n_rows, nr = (n0 + cnt < L ? row0_h[n0 + cnt] : n_rows) - rb;
    const size_t es = esize();
    auto V = [&](void *base) { return (void *)((char *)base + es * n * n0); };  // node n0's vector
    const long long ps0 = (long long)part_stride * n0;
    int k = 0;
    if (ax == AX_OFF) {
        k += project(g, X, true, st, nullptr, 0, 0, false, n0, cnt);
    } else {
        if (ax == AX_REFRESH) k += project(g, X, false, st, AX, g.n_det, 0, false, n0, cnt);
        launch_resid_from_ax(prec, (char *)D + es * (size_t)rb * g.n_det, (char *)AX + es * (size_t)rb * g.n_det,
                             (char *)S + es * (size_t)rb * sp, nr, g.n_det, sp, st);
        k++;
    }
    k += backproject(g, EPI_RESID, R, P, X, st, nullptr, n0, cnt);
    for (int it = 0; it < e1; it++) {
        // ||p||^2 of this step's direction: scal[S_PP] for p0 = r0, then the previous vector
        // pass's per-CTA partials
        const int npp = it == 0 ? 0 : vec_blocks(n);
        k += project(g, P, false, st, nullptr, 0, 0, true, n0, cnt);
        launch_cg_alpha(cnt, scal + (long long)S_NSLOT * n0, cgs + ps0, fp_reduce_blocks(prec, g.n_det), nang + n0,
                        cgp + ps0, npp, cnode + n0, part_stride, st);
        k++;
        if (it + 1 < e1) k += backproject(g, EPI_CGR, R, nullptr, P, st, R, n0, cnt);
        const AxUpdate au{ax == AX_OFF ? nullptr : AX, S, row0 + n0, nang + n0, g.n_det, sp};
        launch_cg_update_px(prec, V(X), V(P), V(R), n, cnt, scal + (long long)S_NSLOT * n0, partial + ps0,
                            part_stride, counter + n0, it + 1 < e1, cgp + ps0, au, st);
        k++;
    }
    return k;
}

// Alg. 2: x <- x - eta (A^T(A x - d) + c x - b'), E1 times
int Inner::gd(const DevGeom &g, int e1, cudaStream_t st) {
    int k = 0;
    for (int it = 0; it < e1; it++) {
        k += project(g, X, true, st);
        k += backproject(g, EPI_GD, X, nullptr, X, st);
    }
    return k;
}

int Inner::norm2(cudaStream_t st) {
    launch_norm2(prec, X, n, L, scal, partial, part_stride, counter, st);
    return 1;
}

// ---------------------------------------------------------------- host geometry
std::vector<AngleHost> make_angles(int n_ang, const double *angles_rad) {
    std::vector<AngleHost> a(n_ang);
    for (int i = 0; i < n_ang; i++) {
        const double th = angles_rad ? angles_rad[i] : M_PI * (double)i / (double)n_ang;
        a[i].cs = cos(th);
        a[i].sn = sin(th);
        if (angles_rad) a[i].xmajor = fabs(a[i].sn) >= fabs(a[i].cs) ? 1 : 0;  // R-3, explicit lists
        else a[i].xmajor = (4 * i >= n_ang && 4 * i <= 3 * n_ang) ? 1 : 0;
        a[i].m = a[i].xmajor ? fabs(a[i].sn) : fabs(a[i].cs);
    }
    return a;
}

void check_angles(const double *angles_rad, int n_ang) {
    if (!angles_rad) return;
    for (int i = 0; i < n_ang; i++)
        TQ_REQUIRE(angles_rad[i] >= 0.0 && angles_rad[i] < M_PI, "angles_rad: every angle must lie in [0, pi)");
}

void partition_angles(int n_ang, int M, int split, std::vector<int> &off, std::vector<int> &idx) {
    off.assign(M + 1, 0);
    idx.clear();
    for (int m = 0; m < M; m++) {
        if (split == TQ_SPLIT_CONTIGUOUS) {
            const int base = n_ang / M, rem = n_ang % M;
            const int start = m * base + std::min(m, rem), cnt = base + (m < rem ? 1 : 0);
            for (int k = 0; k < cnt; k++) idx.push_back(start + k);
        } else {
            for (int a = m; a < n_ang; a += M) idx.push_back(a);
        }
        off[m + 1] = (int)idx.size();
    }
}

void partition_rows(int N, int M, std::vector<int> &row_off) {
    row_off.assign(M + 1, 0);
    const int base = N / M, rem = N % M;
    for (int m = 0; m < M; m++) row_off[m + 1] = row_off[m] + base + (m < rem ? 1 : 0);
}

}  // namespace tq
