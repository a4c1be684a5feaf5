/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Type-generic body of the CPU restatement of the reference hot path. Included twice by
 * coru_oracle.c with T = double (suffix _f64) and T = float (suffix _f32). The fp64
 * instantiation reproduces the reference bit-for-bit when built without FMA contraction
 * (pinned by tests/test_oracle.py against oracle/_ref); the fp32 instantiation is the
 * restatement SURVEY.md §8(c) asks for, since coru::Matrix is fp64-only (matrix.hpp:12).
 *
 * All matrices are dense row-major, like coru::Matrix (matrix.hpp:44-45).
 */
#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SUFFIX)

/* matmul (matrix.hpp:115-131): c(i,.) += a(i,k)·b(k,.) over k increasing. Rows are
 * independent, so the row-parallel split is bit-identical to the serial loop. Four rows share
 * each b(k,.) load (register blocking over i); each entry still sums over k increasing. */
static void FN(mm_)(const T* a, int64_t m, int64_t kk, const T* b, int64_t n, T* c, int threads) {
    memset(c, 0, sizeof(T) * (size_t)(m * n));
    const int64_t mb = (m + 3) / 4;
#pragma omp parallel for schedule(static) num_threads(threads) if (threads > 1 && m > 64)
    for (int64_t ib = 0; ib < mb; ++ib) {
        const int64_t i0 = ib * 4, cnt = m - i0 < 4 ? m - i0 : 4;
        if (cnt < 4) {
            for (int64_t i = i0; i < m; ++i) {
                T* ci = c + i * n;
                const T* ai = a + i * kk;
                for (int64_t k = 0; k < kk; ++k) {
                    const T aik = ai[k];
                    const T* bk = b + k * n;
                    for (int64_t j = 0; j < n; ++j) ci[j] += aik * bk[j];
                }
            }
            continue;
        }
        T *c0 = c + i0 * n, *c1 = c0 + n, *c2 = c1 + n, *c3 = c2 + n;
        const T *a0 = a + i0 * kk, *a1 = a0 + kk, *a2 = a1 + kk, *a3 = a2 + kk;
        for (int64_t k = 0; k < kk; ++k) {
            const T x0 = a0[k], x1 = a1[k], x2 = a2[k], x3 = a3[k];
            const T* bk = b + k * n;
            for (int64_t j = 0; j < n; ++j) {
                const T bj = bk[j];
                c0[j] += x0 * bj;
                c1[j] += x1 * bj;
                c2[j] += x2 * bj;
                c3[j] += x3 * bj;
            }
        }
    }
}

/* matmul(a.transposed(), y) (corutv.hpp:50,57) without materialising a^T: output row j of
 * a^T·y accumulates a(i,j)·y(i,.) over i increasing, exactly the i-k-j order of
 * matmul(at, y); the loop below keeps that per-entry order, so the bits are unchanged.
 * Threads own output rows j; four rows i of a are folded into each accumulator load in
 * sequence ((c + a_i y_i) + a_{i+1} y_{i+1} ...), which is still the serial order. */
static void FN(mm_tn_)(const T* a, int64_t m, int64_t n, const T* y, int64_t d, T* c, int threads) {
    memset(c, 0, sizeof(T) * (size_t)(n * d));
    const int nt = threads > 1 ? threads : 1;
#pragma omp parallel num_threads(nt) if (nt > 1)
    {
#ifdef _OPENMP
        const int t = omp_get_thread_num(), tt = omp_get_num_threads();
#else
        const int t = 0, tt = 1;
#endif
        const int64_t j0 = n * t / tt, j1 = n * (t + 1) / tt;
        int64_t i = 0;
        for (; i + 4 <= m; i += 4) {
            const T *a0 = a + i * n, *a1 = a0 + n, *a2 = a1 + n, *a3 = a2 + n;
            const T *y0 = y + i * d, *y1 = y0 + d, *y2 = y1 + d, *y3 = y2 + d;
            for (int64_t j = j0; j < j1; ++j) {
                const T x0 = a0[j], x1 = a1[j], x2 = a2[j], x3 = a3[j];
                T* cj = c + j * d;
                for (int64_t l = 0; l < d; ++l) {
                    T s = cj[l];
                    s += x0 * y0[l];
                    s += x1 * y1[l];
                    s += x2 * y2[l];
                    s += x3 * y3[l];
                    cj[l] = s;
                }
            }
        }
        for (; i < m; ++i) {
            const T* ai = a + i * n;
            const T* yi = y + i * d;
            for (int64_t j = j0; j < j1; ++j) {
                const T aij = ai[j];
                T* cj = c + j * d;
                for (int64_t l = 0; l < d; ++l) cj[l] += aij * yi[l];
            }
        }
    }
}

/* make_reflector (qr.hpp:32-45) on a column-major working column. */
static T FN(make_reflector_)(int64_t m, int64_t j, T* col) {
    T sigma = 0;
    for (int64_t i = j + 1; i < m; ++i) sigma += col[i] * col[i];
    const T x0 = col[j];
    if (sigma == (T)0) return 0;
    const T mu = SQRT(x0 * x0 + sigma);
    const T v0 = (x0 <= (T)0) ? x0 - mu : -sigma / (x0 + mu);
    const T beta = (T)2 * v0 * v0 / (sigma + v0 * v0);
    for (int64_t i = j + 1; i < m; ++i) col[i] /= v0;
    col[j] = mu;
    return beta;
}

/* apply_reflector (qr.hpp:49-57) */
static void FN(apply_reflector_)(const T* vcol, T beta, int64_t m, int64_t j, T* col) {
    if (beta == (T)0) return;
    T s = col[j];
    for (int64_t i = j + 1; i < m; ++i) s += vcol[i] * col[i];
    s *= beta;
    col[j] -= s;
    for (int64_t i = j + 1; i < m; ++i) col[i] -= s * vcol[i];
}

/* accumulate_q (qr.hpp:60-72) into row-major q (m×n) */
static void FN(accumulate_q_)(const T* w, const T* beta, int64_t m, int64_t n, T* q_out) {
    T* q = (T*)calloc((size_t)(m * n), sizeof(T));
    for (int64_t j = 0; j < n; ++j) q[j * m + j] = 1;
    for (int64_t j = n; j-- > 0;) {
        const T* vcol = w + j * m;
        for (int64_t c = 0; c < n; ++c) FN(apply_reflector_)(vcol, beta[j], m, j, q + c * m);
    }
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) q_out[i * n + j] = q[j * m + i];
    free(q);
}

/* upper_triangle (qr.hpp:74-79) */
static void FN(upper_triangle_)(const T* w, int64_t m, int64_t n, T* r) {
    memset(r, 0, sizeof(T) * (size_t)(n * n));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j && i < n; ++i) r[i * n + j] = w[j * m + i];
}

/* householder_qr (qr.hpp:85-99). Returns 1 (EINVAL) when m < n. `threads` > 1 applies each
 * reflector to the trailing columns (and accumulate_q's columns) in parallel: every column is
 * updated by exactly the reference's loop, so the bits do not depend on the thread count. */
static int FN(householder_qr_mt_)(const T* a, int64_t m, int64_t n, T* q, T* r, int threads) {
    if (m < n || n < 1) return 1;
    T* w = (T*)malloc(sizeof(T) * (size_t)(m * n));
    T* beta = (T*)calloc((size_t)n, sizeof(T));
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) w[j * m + i] = a[i * n + j];
    const int par = threads > 1 && m >= 4096;
    for (int64_t j = 0; j < n; ++j) {
        beta[j] = FN(make_reflector_)(m, j, w + j * m);
        const T* vcol = w + j * m;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) if (par)
        for (int64_t c = j + 1; c < n; ++c) FN(apply_reflector_)(vcol, beta[j], m, j, w + c * m);
    }
    if (q) {
        T* qc = (T*)calloc((size_t)(m * n), sizeof(T));
        for (int64_t j = 0; j < n; ++j) qc[j * m + j] = 1;
        for (int64_t j = n; j-- > 0;) {
            const T* vcol = w + j * m;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) if (par)
            for (int64_t c = 0; c < n; ++c) FN(apply_reflector_)(vcol, beta[j], m, j, qc + c * m);
        }
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) q[i * n + j] = qc[j * m + i];
        free(qc);
    }
    if (r) FN(upper_triangle_)(w, m, n, r);
    free(w);
    free(beta);
    return 0;
}

int FN(oracle_householder_qr_)(const T* a, int64_t m, int64_t n, T* q, T* r) {
    return FN(householder_qr_mt_)(a, m, n, q, r, 1);
}

/* qrcp (qr.hpp:106-143): Businger–Golub, ties to the lowest index (strict >, :122-123),
 * squared-norm downdate with the 1e-6 recompute guard (:133-139). */
int FN(oracle_qrcp_)(const T* a, int64_t m, int64_t n, T* q, T* r, int64_t* perm) {
    if (m < n || n < 1) return 1;
    T* w = (T*)malloc(sizeof(T) * (size_t)(m * n));
    T* beta = (T*)calloc((size_t)n, sizeof(T));
    T* colsq = (T*)malloc(sizeof(T) * (size_t)n);
    T* base = (T*)malloc(sizeof(T) * (size_t)n);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) w[j * m + i] = a[i * n + j];
    for (int64_t j = 0; j < n; ++j) perm[j] = j;
    for (int64_t j = 0; j < n; ++j) {
        T s = 0;
        for (int64_t i = 0; i < m; ++i) s += w[j * m + i] * w[j * m + i];
        colsq[j] = base[j] = s;
    }
    for (int64_t j = 0; j < n; ++j) {
        int64_t piv = j;
        for (int64_t c = j + 1; c < n; ++c)
            if (colsq[c] > colsq[piv]) piv = c;
        if (piv != j) {
            for (int64_t i = 0; i < m; ++i) {
                T x = w[j * m + i]; w[j * m + i] = w[piv * m + i]; w[piv * m + i] = x;
            }
            T x = colsq[j]; colsq[j] = colsq[piv]; colsq[piv] = x;
            x = base[j]; base[j] = base[piv]; base[piv] = x;
            int64_t p = perm[j]; perm[j] = perm[piv]; perm[piv] = p;
        }
        beta[j] = FN(make_reflector_)(m, j, w + j * m);
        const T* vcol = w + j * m;
        for (int64_t c = j + 1; c < n; ++c) {
            FN(apply_reflector_)(vcol, beta[j], m, j, w + c * m);
            colsq[c] -= w[c * m + j] * w[c * m + j];
            if (colsq[c] < (T)1e-6 * base[c]) {
                T s = 0;
                for (int64_t i = j + 1; i < m; ++i) s += w[c * m + i] * w[c * m + i];
                colsq[c] = base[c] = s;
            }
        }
    }
    if (q) FN(accumulate_q_)(w, beta, m, n, q);
    if (r) FN(upper_triangle_)(w, m, n, r);
    free(w); free(beta); free(colsq); free(base);
    return 0;
}

/* detail::sketch_bases (corutv.hpp:49-65). q1 m×ell, q2 n×ell, c1 m×ell, c2_prev n×ell
 * (any output may be NULL). */
int FN(oracle_sketch_bases_)(const T* a, int64_t m, int64_t n, int64_t ell, int q, uint64_t seed,
                             uint64_t stream, int threads, T* q1, T* q2, T* c1_out, T* c2p_out,
                             int* warn) {
    if (ell < 1 || ell >= (m < n ? m : n) || q < 0) return 1;
    T* c2 = (T*)malloc(sizeof(T) * (size_t)(n * ell));
    T* c2p = (T*)malloc(sizeof(T) * (size_t)(n * ell));
    T* c1 = (T*)malloc(sizeof(T) * (size_t)(m * ell));
    T* r1 = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
    /* Φ = gaussian(n, ell, seed) (corutv.hpp:51); fp32 rounds the fp64 stream. */
    double* phi = (double*)malloc(sizeof(double) * (size_t)(n * ell));
    oracle_gaussian(n, ell, seed, stream, phi);
    for (int64_t i = 0; i < n * ell; ++i) c2[i] = (T)phi[i];
    free(phi);
    for (int i = 0; i <= q; ++i) {
        FN(mm_)(a, m, n, c2, ell, c1, threads);     /* c1 = a·c2 (corutv.hpp:55) */
        memcpy(c2p, c2, sizeof(T) * (size_t)(n * ell)); /* c2_prev (corutv.hpp:56) */
        FN(mm_tn_)(a, m, n, c1, ell, c2, threads);  /* c2 = a^T·c1 (corutv.hpp:57) */
    }
    FN(householder_qr_mt_)(c1, m, ell, q1, r1, threads);
    if (q2) FN(householder_qr_mt_)(c2, n, ell, q2, NULL, threads);
    const double r00 = fabs((double)r1[0]);
    const double rll = fabs((double)r1[(ell - 1) * ell + (ell - 1)]);
    if (warn) *warn = rll <= 1e-14 * r00;
    if (c1_out) memcpy(c1_out, c1, sizeof(T) * (size_t)(m * ell));
    if (c2p_out) memcpy(c2p_out, c2p, sizeof(T) * (size_t)(n * ell));
    free(c2); free(c2p); free(c1); free(r1);
    return 0;
}

/* corutv (corutv.hpp:79-100), variant 0 = DVariant::exact, 1 = DVariant::approx.
 * u m×ell, t ell×ell, v n×ell; flags[0] = lower, flags[1] = conditioning_warning, perm_out
 * (optional) = QRCP pivots. Returns 1 for the reference's std::invalid_argument cases.
 * approx (corutv.hpp:91-92): d = (q1^T·c1)·pinv(q2^T·c2_prev); the pinv (Jacobi SVD, svd.hpp)
 * runs in fp64 for both instantiations (the reference's tolerances are fp64 constants) and is
 * rounded to T; the two products around it run in T. */
int FN(oracle_corutv_)(const T* a, int64_t m, int64_t n, int64_t ell, int q, int variant,
                       uint64_t seed, uint64_t stream, int threads, T* u, T* t, T* v, int* flags,
                       int64_t* perm_out) {
    if (ell < 1 || ell >= (m < n ? m : n) || q < 0) return 1;
    if (variant != 0 && variant != 1) return 1;
    if (m < n) {
        /* corutv(a^T) and swap (corutv.hpp:82-87) */
        T* at = (T*)malloc(sizeof(T) * (size_t)(m * n));
        for (int64_t i = 0; i < m; ++i)
            for (int64_t j = 0; j < n; ++j) at[j * m + i] = a[i * n + j];
        T* tt = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
        int rc = FN(oracle_corutv_)(at, n, m, ell, q, variant, seed, stream, threads, v, tt, u, flags, perm_out);
        for (int64_t i = 0; i < ell; ++i)
            for (int64_t j = 0; j < ell; ++j) t[i * ell + j] = tt[j * ell + i];
        flags[0] = 1;
        free(at); free(tt);
        return rc;
    }
    T* q1 = (T*)malloc(sizeof(T) * (size_t)(m * ell));
    T* q2 = (T*)malloc(sizeof(T) * (size_t)(n * ell));
    int warn = 0;
    T* d = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
    T* q1ta = NULL;
    if (variant == 1) {
        T* c1 = (T*)malloc(sizeof(T) * (size_t)(m * ell));
        T* c2p = (T*)malloc(sizeof(T) * (size_t)(n * ell));
        FN(oracle_sketch_bases_)(a, m, n, ell, q, seed, stream, threads, q1, q2, c1, c2p, &warn);
        T* y1 = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
        T* y2 = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
        FN(mm_tn_)(q1, m, ell, c1, ell, y1, threads);  /* q1^T·c1: matmul(q1.transposed(), c1) */
        FN(mm_tn_)(q2, n, ell, c2p, ell, y2, threads); /* q2^T·c2_prev */
        double* yd = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
        double* pd = (double*)malloc(sizeof(double) * (size_t)(ell * ell));
        for (int64_t i = 0; i < ell * ell; ++i) yd[i] = (double)y2[i];
        oracle_pinv_f64(yd, ell, pd);
        for (int64_t i = 0; i < ell * ell; ++i) y2[i] = (T)pd[i];
        FN(mm_)(y1, ell, ell, y2, ell, d, 1);          /* (q1^T c1)·pinv(q2^T c2_prev) */
        free(c1); free(c2p); free(y1); free(y2); free(yd); free(pd);
    } else {
        FN(oracle_sketch_bases_)(a, m, n, ell, q, seed, stream, threads, q1, q2, NULL, NULL, &warn);
        /* d = (q1^T·a)·q2 (corutv.hpp:90): q1^T·a is the tn product of (a-as-m×n, q1). Its row l
         * accumulates q1(i,l)·a(i,.) over i increasing — matmul(q1.transposed(), a)'s order. */
        q1ta = (T*)calloc((size_t)(ell * n), sizeof(T));
        /* threads split the columns j: each entry still sums over i increasing, and A is read
         * once instead of once per row l */
        const int nt = threads > 1 ? threads : 1;
#pragma omp parallel num_threads(nt) if (nt > 1)
        {
#ifdef _OPENMP
            const int th = omp_get_thread_num(), tt = omp_get_num_threads();
#else
            const int th = 0, tt = 1;
#endif
            const int64_t j0 = n * th / tt, j1 = n * (th + 1) / tt;
            int64_t i = 0;
            for (; i + 4 <= m; i += 4) {  /* four rows of a folded in sequence per load */
                const T *a0 = a + i * n, *a1 = a0 + n, *a2 = a1 + n, *a3 = a2 + n;
                for (int64_t l = 0; l < ell; ++l) {
                    const T w0 = q1[i * ell + l], w1 = q1[(i + 1) * ell + l];
                    const T w2 = q1[(i + 2) * ell + l], w3 = q1[(i + 3) * ell + l];
                    T* row = q1ta + l * n;
                    for (int64_t j = j0; j < j1; ++j) {
                        T s = row[j];
                        s += w0 * a0[j];
                        s += w1 * a1[j];
                        s += w2 * a2[j];
                        s += w3 * a3[j];
                        row[j] = s;
                    }
                }
            }
            for (; i < m; ++i) {
                const T* ai = a + i * n;
                for (int64_t l = 0; l < ell; ++l) {
                    const T w = q1[i * ell + l];
                    T* row = q1ta + l * n;
                    for (int64_t j = j0; j < j1; ++j) row[j] += w * ai[j];
                }
            }
        }
        FN(mm_)(q1ta, ell, n, q2, ell, d, 1);
    }
    T* qm = (T*)malloc(sizeof(T) * (size_t)(ell * ell));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)ell);
    FN(oracle_qrcp_)(d, ell, ell, qm, t, perm);          /* corutv.hpp:93 */
    FN(mm_)(q1, m, ell, qm, ell, u, threads);            /* u = q1·Q (corutv.hpp:94) */
    for (int64_t j = 0; j < ell; ++j)                    /* v(:,j) = q2(:,perm[j]) (:95-97) */
        for (int64_t i = 0; i < n; ++i) v[i * ell + j] = q2[i * ell + perm[j]];
    if (perm_out) memcpy(perm_out, perm, sizeof(int64_t) * (size_t)ell);
    flags[0] = 0;
    flags[1] = warn;
    free(q1); free(q2); free(q1ta); free(d); free(qm); free(perm);
    return 0;
}

/* matmul exposed for kernel-level parity (matrix.hpp:115-131). */
int FN(oracle_matmul_)(const T* a, int64_t m, int64_t k, const T* b, int64_t n, T* c, int threads) {
    FN(mm_)(a, m, k, b, n, c, threads);
    return 0;
}

/* matmul(a.transposed(), y) as used at corutv.hpp:57. */
int FN(oracle_matmul_tn_)(const T* a, int64_t m, int64_t n, const T* y, int64_t d, T* c, int threads) {
    FN(mm_tn_)(a, m, n, y, d, c, threads);
    return 0;
}

#undef FN
#undef CAT
#undef CAT_
