/*
 * bagel_oracle.c -- plain, slow, float64 CPU oracle for BAGEL's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2202_13638_b200/csrc); neither includes the other.
 *
 * Passages followed (PAPER.md = P:line, SPEC.md = S:line):
 *   SE-ARD kernel ............ Eq.4, P:72-76 (Lambda = diag(l^-2), reading R1)
 *   exact posterior .......... Eq.2-3, P:67-71 (prior mean 0, latent variance)
 *   LOVE cache / variance .... P:46, P:81 (Lanczos on Khat, R = L_T^-1 Q^T; R20)
 *   policy ................... P:104, P:129, P:149 (tanh MLP, bounded output)
 *   GP transition sample ..... Eq.9-10, P:130-138 (x' = x + mu + sigma*eps, Delta targets)
 *   reward / return / loss ... Eq.7-8; Alg.1 lines P:101-108
 *   gradient ................. Alg.1 "Compute grad_theta L via Autodiff", P:109 --
 *                              written out as hand reverse mode, pinned by central FD.
 *   Philox4x32-10 ............ Salmon et al. (SC'11) Random123 definition; DESIGN.md "Philox".
 *
 * Every routine is the definition written out, in the paper's order, in
 * float64.  No blocking, no fusion.  Loops over independent trajectories /
 * rows may run under OpenMP; every reduction is done in a fixed order so the
 * result does not depend on the thread count.
 *
 * Pins (tests/test_oracle_*.py): Philox KATs; kernel special values; N=1 and
 * N=2 closed forms; Gauss-Jordan brute-force inverses at N<=8; LOVE rank N ==
 * exact variance; Galerkin monotonicity in rank; interpolation / far-field
 * limits; constant-kernel closed form; scalar rollout closed form; reward
 * values of S:388; central-FD gradient.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_VAR_FLOOR 1e-12 /* S:252 clamp, reading R19 */

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Random123).  round: {hi1^c1^k0, lo1, hi0^c3^k1, lo0} */
/* ------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { /* key schedule: bump between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 23-bit uniform strictly inside (0,1): ((o >> 9) + 0.5) * 2^-23.  Every value
 * has at most 24 significant bits, so it is exact in fp32 and fp64 alike
 * (reading R29). */
static double orc_uniform(uint32_t o) { return ((double)(o >> 9) + 0.5) * (1.0 / 8388608.0); }

/* Box-Muller on the four uniforms of one Philox call (fp64). */
void orc_box_muller4(const uint32_t o[4], double eps[4])
{
    double u0 = orc_uniform(o[0]), u1 = orc_uniform(o[1]);
    double u2 = orc_uniform(o[2]), u3 = orc_uniform(o[3]);
    const double two_pi = 6.283185307179586476925286766559;
    double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u2));
    eps[0] = r0 * cos(two_pi * u1);
    eps[1] = r0 * sin(two_pi * u1);
    eps[2] = r1 * cos(two_pi * u3);
    eps[3] = r1 * sin(two_pi * u3);
}

/* Rollout noise eps_{b,t,m}: key = (seed lo, seed hi), ctr = (b_global, t, m>>2, 0). */
double orc_rollout_eps(uint64_t seed, uint32_t b_global, uint32_t t, int m)
{
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {b_global, t, (uint32_t)(m >> 2), 0u};
    uint32_t o[4];
    double e[4];
    orc_philox4x32_10(ctr, key, o);
    orc_box_muller4(o, e);
    return e[m & 3];
}

/* Lanczos restart vector component n: key = ("LOVE", 0), ctr = (restart_idx, n>>2, m, 1). */
static double orc_restart_component(uint32_t restart_idx, int n, int m)
{
    uint32_t key[2] = {0x4C4F5645u, 0u};
    uint32_t ctr[4] = {restart_idx, (uint32_t)(n >> 2), (uint32_t)m, 1u};
    uint32_t o[4];
    double e[4];
    orc_philox4x32_10(ctr, key, o);
    orc_box_muller4(o, e);
    return e[n & 3];
}

/* ------------------------------------------------------------------ */
/* Eq.4: k(a,b) = s * exp(-1/2 sum_c (a_c - b_c)^2 / l_c^2)            */
/* ------------------------------------------------------------------ */
double orc_kernel(const double* a, const double* b, int d, const double* ell, double s)
{
    double q = 0.0;
    for (int c = 0; c < d; ++c) {
        double diff = a[c] - b[c];
        q += diff * diff / (ell[c] * ell[c]);
    }
    return s * exp(-0.5 * q);
}

void orc_kernel_matrix(const double* A, int na, const double* B, int nb, int d,
                       const double* ell, double s, double* K /* na x nb */)
{
    for (int i = 0; i < na; ++i)
        for (int j = 0; j < nb; ++j)
            K[(size_t)i * nb + j] = orc_kernel(A + (size_t)i * d, B + (size_t)j * d, d, ell, s);
}

/* Khat = K(X,X) + noise * I */
static double* orc_khat(const double* X, int N, int d, const double* ell, double s, double noise)
{
    double* K = (double*)malloc(sizeof(double) * (size_t)N * N);
    if (!K) return NULL;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < N; ++i) {
        for (int j = 0; j < N; ++j)
            K[(size_t)i * N + j] = orc_kernel(X + (size_t)i * d, X + (size_t)j * d, d, ell, s);
        K[(size_t)i * N + i] += noise;
    }
    return K;
}

/* Cholesky-Crout, in place, lower triangle of row-major A (upper set to 0).
 * Returns 0 on success, else (pivot index + 1) of the first pivot <= 0 (DESIGN R27). */
int orc_cholesky(double* A, int n)
{
    for (int j = 0; j < n; ++j) {
        double* Lj = A + (size_t)j * n;
        double djj = Lj[j];
        for (int k = 0; k < j; ++k) djj -= Lj[k] * Lj[k];
        if (!(djj > 0.0)) return j + 1;
        double ljj = sqrt(djj);
        Lj[j] = ljj;
#pragma omp parallel for schedule(static) if (n - j > 256)
        for (int i = j + 1; i < n; ++i) {
            double* Li = A + (size_t)i * n;
            double v = Li[j];
            for (int k = 0; k < j; ++k) v -= Li[k] * Lj[k];
            Li[j] = v / ljj;
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = 0.0;
    return 0;
}

/* L x = b (forward), then optionally L^T x = (.) (backward); L lower, row-major. */
static void orc_forward_solve(const double* L, int n, const double* b, double* x)
{
    for (int i = 0; i < n; ++i) {
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= L[(size_t)i * n + k] * x[k];
        x[i] = v / L[(size_t)i * n + i];
    }
}
static void orc_backward_solve_T(const double* L, int n, const double* b, double* x)
{
    for (int i = n - 1; i >= 0; --i) {
        double v = b[i];
        for (int k = i + 1; k < n; ++k) v -= L[(size_t)k * n + i] * x[k];
        x[i] = v / L[(size_t)i * n + i];
    }
}

/* Exact GP cache for one output: L = chol(Khat), alpha = Khat^-1 y (Eq.2).
 * L_out may be NULL.  Returns 0 or pivot+1. */
int orc_exact_fit(const double* X, int N, int d, const double* y, const double* ell, double s,
                  double noise, double* alpha_out, double* L_out)
{
    double* K = orc_khat(X, N, d, ell, s, noise);
    if (!K) return -1;
    int rc = orc_cholesky(K, N);
    if (rc == 0) {
        double* tmp = (double*)malloc(sizeof(double) * N);
        orc_forward_solve(K, N, y, tmp);
        orc_backward_solve_T(K, N, tmp, alpha_out);
        free(tmp);
        if (L_out) memcpy(L_out, K, sizeof(double) * (size_t)N * N);
    }
    free(K);
    return rc;
}

/* Eq.2-3 exact: mean = k^T alpha, var = s - ||L^-1 k||^2 (no clamp). */
void orc_exact_predict(const double* X, int N, int d, const double* ell, double s,
                       const double* L, const double* alpha, const double* xs, int M,
                       double* mean, double* var)
{
#pragma omp parallel for schedule(static)
    for (int i = 0; i < M; ++i) {
        double* kv = (double*)malloc(sizeof(double) * N);
        double* v = (double*)malloc(sizeof(double) * N);
        const double* x = xs + (size_t)i * d;
        double mu = 0.0;
        for (int n = 0; n < N; ++n) {
            kv[n] = orc_kernel(x, X + (size_t)n * d, d, ell, s);
            mu += kv[n] * alpha[n];
        }
        orc_forward_solve(L, N, kv, v);
        double q = 0.0;
        for (int n = 0; n < N; ++n) q += v[n] * v[n];
        mean[i] = mu;
        var[i] = orc_kernel(x, x, d, ell, s) - q;
        free(kv);
        free(v);
    }
}

/* ------------------------------------------------------------------ */
/* LOVE cache (recipe = DESIGN.md reading R20):            */
/*   q1 = y/||y||; k Lanczos steps on Khat with classical Gram-Schmidt */
/*   against all previous q, twice; breakdown b_j <= 1e-10 max|a_i|    */
/*   -> restart with a Philox vector; T = tridiag(a,b); L_T = chol(T); */
/*   R = L_T^-1 Q^T (k x N).  Khat^-1 ~= R^T R.                         */
/* Returns 0, or -(j+1) if T is not PD at row j, or -1000 on OOM.       */
/* ------------------------------------------------------------------ */
static void orc_gs_twice(const double* Qm, int nq, int N, double* v)
{
    double* c = (double*)malloc(sizeof(double) * (nq > 0 ? nq : 1));
    for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i < nq; ++i) { /* c = Q^T v (all from the same v: classical GS) */
            double acc = 0.0;
            for (int n = 0; n < N; ++n) acc += Qm[(size_t)i * N + n] * v[n];
            c[i] = acc;
        }
        for (int n = 0; n < N; ++n) { /* v -= Q c */
            double acc = 0.0;
            for (int i = 0; i < nq; ++i) acc += Qm[(size_t)i * N + n] * c[i];
            v[n] -= acc;
        }
    }
    free(c);
}

static double orc_norm(const double* v, int N)
{
    double acc = 0.0;
    for (int n = 0; n < N; ++n) acc += v[n] * v[n];
    return sqrt(acc);
}

int orc_love_build(const double* X, int N, int d, const double* y, const double* ell, double s,
                   double noise, int m_index, int k, double* R_out /* k x N */,
                   double* a_out /* k, nullable */, double* b_out /* k-1, nullable */,
                   int* restarts_out)
{
    double* K = orc_khat(X, N, d, ell, s, noise);
    double* Qm = (double*)calloc((size_t)k * N, sizeof(double)); /* rows q_0..q_{k-1} */
    double* v = (double*)malloc(sizeof(double) * N);
    double* a = (double*)malloc(sizeof(double) * k);
    double* b = (double*)calloc(k, sizeof(double));
    if (!K || !Qm || !v || !a || !b) return -1000;
    uint32_t restart_idx = 0;

    double ny = orc_norm(y, N);
    if (ny > 0.0) {
        for (int n = 0; n < N; ++n) Qm[n] = y[n] / ny;
    } else { /* restart vector for a zero probe */
        for (int n = 0; n < N; ++n) v[n] = orc_restart_component(restart_idx, n, m_index);
        restart_idx++;
        double nv = orc_norm(v, N);
        for (int n = 0; n < N; ++n) Qm[n] = v[n] / nv;
    }
    double amax = 0.0;
    for (int j = 0; j < k; ++j) {
        const double* qj = Qm + (size_t)j * N;
        /* v = Khat q_j */
#pragma omp parallel for schedule(static) if (N > 256)
        for (int i = 0; i < N; ++i) {
            double acc = 0.0;
            for (int n = 0; n < N; ++n) acc += K[(size_t)i * N + n] * qj[n];
            v[i] = acc;
        }
        double aj = 0.0;
        for (int n = 0; n < N; ++n) aj += qj[n] * v[n];
        a[j] = aj;
        if (fabs(aj) > amax) amax = fabs(aj);
        orc_gs_twice(Qm, j + 1, N, v);
        double bj = orc_norm(v, N);
        if (j < k - 1) {
            double* qn = Qm + (size_t)(j + 1) * N;
            if (bj <= 1e-10 * amax) { /* breakdown: deterministic Philox restart */
                for (int n = 0; n < N; ++n) v[n] = orc_restart_component(restart_idx, n, m_index);
                restart_idx++;
                orc_gs_twice(Qm, j + 1, N, v);
                double nv = orc_norm(v, N);
                for (int n = 0; n < N; ++n) qn[n] = v[n] / nv;
                b[j] = 0.0;
            } else {
                for (int n = 0; n < N; ++n) qn[n] = v[n] / bj;
                b[j] = bj;
            }
        }
    }
    /* L_T = chol(T): lower bidiagonal (diag l_j, sub-diag e_j) */
    double* ld = (double*)malloc(sizeof(double) * k);
    double* le = (double*)calloc(k, sizeof(double));
    int rc = 0;
    for (int j = 0; j < k; ++j) {
        double dj = a[j];
        if (j > 0) {
            le[j] = b[j - 1] / ld[j - 1];
            dj -= le[j] * le[j];
        }
        if (!(dj > 0.0)) { rc = -(j + 1); break; }
        ld[j] = sqrt(dj);
    }
    if (rc == 0) {
        /* R = L_T^-1 Q^T: forward substitution, row by row */
        for (int j = 0; j < k; ++j)
            for (int n = 0; n < N; ++n) {
                double v0 = Qm[(size_t)j * N + n];
                if (j > 0) v0 -= le[j] * R_out[(size_t)(j - 1) * N + n];
                R_out[(size_t)j * N + n] = v0 / ld[j];
            }
    }
    if (a_out) memcpy(a_out, a, sizeof(double) * k);
    if (b_out && k > 1) memcpy(b_out, b, sizeof(double) * (k - 1));
    if (restarts_out) *restarts_out = (int)restart_idx;
    free(K); free(Qm); free(v); free(a); free(b); free(ld); free(le);
    return rc;
}

/* ------------------------------------------------------------------ */
/* One GP query with LOVE variance and input Jacobians (Appendix B):   */
/*   k_n = s exp(...), mu = k.alpha, z = R k, v = s - ||z||^2,          */
/*   Jmu_c = (1/l_c^2) sum_n k_n alpha_n (X_nc - x*_c),                 */
/*   w = R^T z, Jv_c = (2/l_c^2) sum_n w_n k_n (x*_c - X_nc).           */
/* Also returns the conditioning terms used by the parity tolerances:   */
/*   mbound = sum_n |k_n alpha_n|,  vbound = 2 sum_j |z_j| sum_n |R_jn k_n|. */
/* scratch: 2N + k doubles.                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int N, d, p, k;
    const double* X;     /* N x d */
    const double* ell;   /* p x d */
    const double* s;     /* p */
    const double* alpha; /* p x N   (Khat^-1 y, not scaled by s) */
    const double* R;     /* p x k x N */
    int abs_target;      /* 0: Delta targets x' = x + f (R6); 1: absolute x' = f (NEXT-4) */
} orc_gp;

/* fp32-sensitivity mode (variant (a)): every kernel value entering the
 * mean path (mu, J^mu; mode 1 or 2) and/or the variance path (z, J^v; mode 1 or 3) is
 * multiplied by (1 + delta), delta ~ U(-2^-22, 2^-22) from a Philox stream keyed by `seed`
 * with counter (b_global, t, m * N + n, 5 | 6).  It measures the parity floor any fp32
 * implementation can reach on a problem; mode 0 is the exact oracle. */
typedef struct {
    int mode;
    uint64_t seed;
    uint32_t b, t;
} orc_perturb;

static double orc_delta(const orc_perturb* pt, int m, int N, int n, uint32_t stream)
{
    uint32_t key[2] = {(uint32_t)(pt->seed & 0xffffffffu), (uint32_t)(pt->seed >> 32)};
    uint32_t ctr[4] = {pt->b, pt->t, (uint32_t)(m * N + n), stream};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return (orc_uniform(o[0]) * 2.0 - 1.0) * (1.0 / 4194304.0); /* U(-2^-22, 2^-22) */
}

static void orc_query_p(const orc_gp* gp, int m, const double* x, double* scratch, double* mean,
                        double* var, double* jmu, double* jv, double* mbound, double* vbound,
                        const orc_perturb* pt)
{
    const int N = gp->N, d = gp->d, k = gp->k;
    const double* ell = gp->ell + (size_t)m * d;
    const double s = gp->s[m];
    const double* alpha = gp->alpha + (size_t)m * N;
    const double* R = gp->R + (size_t)m * k * N;
    double* kv = scratch;              /* kernel values of the mean path */
    double* w = scratch + N;
    double* z = scratch + 2 * N;
    double* kvv = scratch + 2 * N + k; /* kernel values of the variance path */
    const int pm = pt ? pt->mode : 0;
    double mu = 0.0, mb = 0.0;
    for (int n = 0; n < N; ++n) {
        double kn = orc_kernel(x, gp->X + (size_t)n * d, d, ell, s);
        if (pm == 4 || pm == 5) {
            /* variant (b): the exponent as an fp32 GPU forms it -- mode 4 scales before the
             * difference (x_hat - X_hat with x_hat = fl(x kappa/l)), mode 5 differences first
             * then scales; exp2 and everything else exact. */
            const float kap = 0.84932180028801907f;
            float q = 0.0f;
            for (int c = 0; c < d; ++c) {
                const float sc = (float)((double)kap / ell[c]);
                float df;
                if (pm == 4) {
                    const float xh = (float)x[c] * sc, Xh = (float)gp->X[(size_t)n * d + c] * sc;
                    df = xh - Xh;
                } else {
                    df = ((float)x[c] - (float)gp->X[(size_t)n * d + c]) * sc;
                }
                q = fmaf(df, df, q);
            }
            kn = s * exp2(-(double)q);
        }
        kv[n] = (pm == 1 || pm == 2) ? kn * (1.0 + orc_delta(pt, m, N, n, 5)) : kn;  /* mode 4/5: kn above */
        kvv[n] = (pm == 1 || pm == 3) ? kn * (1.0 + orc_delta(pt, m, N, n, 6)) : kn;
        mu += kv[n] * alpha[n];
        mb += fabs(kv[n] * alpha[n]);
    }
    double zz = 0.0, vb = 0.0;
    for (int j = 0; j < k; ++j) {
        double acc = 0.0, aabs = 0.0;
        for (int n = 0; n < N; ++n) {
            acc += R[(size_t)j * N + n] * kvv[n];
            aabs += fabs(R[(size_t)j * N + n] * kvv[n]);
        }
        z[j] = acc;
        zz += acc * acc;
        vb += 2.0 * fabs(acc) * aabs;
    }
    *mean = mu;
    *var = s - zz; /* k(x*,x*) = s */
    if (mbound) *mbound = mb;
    if (vbound) *vbound = vb;
    if (jmu || jv) {
        for (int n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int j = 0; j < k; ++j) acc += R[(size_t)j * N + n] * z[j];
            w[n] = acc;
        }
        for (int c = 0; c < d; ++c) {
            double il2 = 1.0 / (ell[c] * ell[c]);
            double am = 0.0, av = 0.0;
            for (int n = 0; n < N; ++n) {
                double dx = gp->X[(size_t)n * d + c] - x[c];
                am += kv[n] * alpha[n] * dx;
                av += w[n] * kvv[n] * (-dx);
            }
            if (jmu) jmu[c] = il2 * am;
            if (jv) jv[c] = 2.0 * il2 * av;
        }
    }
}

static void orc_query(const orc_gp* gp, int m, const double* x, double* scratch, double* mean,
                      double* var, double* jmu, double* jv, double* mbound, double* vbound)
{
    orc_query_p(gp, m, x, scratch, mean, var, jmu, jv, mbound, vbound, NULL);
}

/* Batched query for all outputs: outputs are M x p (mean, var, bounds) and M x p x d (Jacobians). */
void orc_love_predict(const orc_gp* gp, const double* xs, int M, double* mean, double* var,
                      double* jmu, double* jv, double* mbound, double* vbound)
{
    const int p = gp->p, d = gp->d;
#pragma omp parallel
    {
        double* scratch = (double*)malloc(sizeof(double) * (3 * (size_t)gp->N + gp->k + 1));
#pragma omp for schedule(static)
        for (int i = 0; i < M; ++i)
            for (int m = 0; m < p; ++m) {
                size_t o = (size_t)i * p + m;
                orc_query(gp, m, xs + (size_t)i * d, scratch, mean + o, var + o,
                          jmu ? jmu + o * d : NULL, jv ? jv + o * d : NULL,
                          mbound ? mbound + o : NULL, vbound ? vbound + o : NULL);
            }
        free(scratch);
    }
}

/* ------------------------------------------------------------------ */
/* Policy: h0 = phi(x, g); h_l = tanh(W_l h + b_l) */
/* theta layout: per layer W_l [out x in] row-major, then b_l [out].     */
/* phi_mode 0: [x, g] (in = 2p);  1: [x, g, g - x] (in = 3p).             */
/* ------------------------------------------------------------------ */
typedef struct {
    int n_layers;
    const int* sizes;    /* n_layers + 1 */
    int phi_mode;
    const double* theta;
} orc_policy;

typedef struct {
    const double* Q;     /* p (diagonal) */
    double sigma_r;
} orc_reward;

static int orc_max_width(const orc_policy* pol)
{
    int w = 0;
    for (int l = 0; l <= pol->n_layers; ++l)
        if (pol->sizes[l] > w) w = pol->sizes[l];
    return w;
}

/* h: (n_layers+1) x maxw activations (h[0] = phi(x,g)). */
static void orc_mlp_forward(const orc_policy* pol, int p, const double* x, const double* g, double* h,
                            int maxw)
{
    for (int c = 0; c < p; ++c) {
        h[c] = x[c];
        h[p + c] = g[c];
        if (pol->phi_mode == 1) h[2 * p + c] = g[c] - x[c];
    }
    const double* th = pol->theta;
    for (int l = 0; l < pol->n_layers; ++l) {
        int in = pol->sizes[l], out = pol->sizes[l + 1];
        const double* W = th;
        const double* b = th + (size_t)in * out;
        const double* hi = h + (size_t)l * maxw;
        double* ho = h + (size_t)(l + 1) * maxw;
        for (int o = 0; o < out; ++o) {
            double a = b[o];
            for (int i = 0; i < in; ++i) a += W[(size_t)o * in + i] * hi[i];
            ho[o] = tanh(a);
        }
        th += (size_t)in * out + out;
    }
}

/* Test export of the policy forward above: u_b = pi(x_b, g_b) for B rows (R13/R14),
 * u is B x sizes[n_layers].  Pinned against torch.nn.Sequential in tests/test_oracle_rollout.py. */
void orc_policy_act(const orc_policy* pol, int p, const double* x, const double* g, int B, double* u)
{
    const int maxw = orc_max_width(pol), q = pol->sizes[pol->n_layers];
    double* h = (double*)malloc(sizeof(double) * (size_t)(pol->n_layers + 1) * maxw);
    for (int b = 0; b < B; ++b) {
        orc_mlp_forward(pol, p, x + (size_t)b * p, g + (size_t)b * p, h, maxw);
        for (int o = 0; o < q; ++o) u[(size_t)b * q + o] = h[(size_t)pol->n_layers * maxw + o];
    }
    free(h);
}

/* Eq.8: r = exp(-(1/(2 sigma_r^2)) sum_c Q_c (x_c - g_c)^2) */
double orc_reward_fn(const orc_reward* rw, int p, const double* x, const double* g)
{
    double q = 0.0;
    for (int c = 0; c < p; ++c) q += rw->Q[c] * (x[c] - g[c]) * (x[c] - g[c]);
    return exp(-q / (2.0 * rw->sigma_r * rw->sigma_r));
}

/* ------------------------------------------------------------------ */
/* Rollout (Alg.1 P:101-108 with Eq.9-11) and its exact gradient.       */
/* cost_out = -(1/B_global) sum_b sum_{t=0}^{T} r_{b,t}  (this shard).  */
/* grad_out = d cost / d theta (this shard's contribution).             */
/* eps_mode: 0 = Philox (seed, traj_offset+b, t, m); 1 = zero noise.   */
/* Traces (nullable): xs (T+1) x B x p, mu/var T x B x p, ret B.        */
/* Returns 0, or 1 + (t * B + b) of the first non-finite state.        */
/* ------------------------------------------------------------------ */
int orc_rollout(const orc_gp* gp, const orc_policy* pol, const orc_reward* rw, const double* x0,
                const double* goals, int B, int T, uint64_t seed, long long traj_offset,
                long long B_global, int eps_mode, int want_grad, double* cost_out,
                double* grad_out, double* trace_x, double* trace_mu, double* trace_var,
                double* ret_out, int perturb_mode, uint64_t perturb_seed)
{
    const int p = gp->p, d = gp->d, L = pol->n_layers;
    const int maxw = orc_max_width(pol);
    size_t n_theta = 0;
    for (int l = 0; l < L; ++l) n_theta += (size_t)(pol->sizes[l] + 1) * pol->sizes[l + 1];
    const double invB = 1.0 / (double)B_global;
    double* ret = (double*)calloc(B, sizeof(double));
    double* gper = want_grad ? (double*)calloc((size_t)B * n_theta, sizeof(double)) : NULL;
    int bad = 0;

#pragma omp parallel
    {
        double* scratch = (double*)malloc(sizeof(double) * (3 * (size_t)gp->N + gp->k + 1));
        /* per-trajectory tape */
        double* tx = (double*)malloc(sizeof(double) * (size_t)(T + 1) * p);
        double* th = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * (L + 1) * maxw);
        double* tjm = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * p * d);
        double* tjv = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * p * d);
        double* tsig = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * p);
        double* tvpos = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * p);
        double* teps = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1) * p);
        double* xs = (double*)malloc(sizeof(double) * d);
        double* hbar = (double*)malloc(sizeof(double) * 2 * maxw);
        double* xbar = (double*)malloc(sizeof(double) * p);
        double* xsbar = (double*)malloc(sizeof(double) * d);

#pragma omp for schedule(static)
        for (int b = 0; b < B; ++b) {
            const double* g = goals + (size_t)b * p;
            const uint32_t bg = (uint32_t)(traj_offset + b);
            for (int c = 0; c < p; ++c) tx[c] = x0[(size_t)b * p + c];
            double G = orc_reward_fn(rw, p, tx, g); /* Alg.1: G <- r(S0, G) */
            if (trace_x)
                for (int c = 0; c < p; ++c) trace_x[(size_t)b * p + c] = tx[c];
            int dead = 0;
            for (int t = 0; t < T && !dead; ++t) {
                const double* x = tx + (size_t)t * p;
                double* h = th + (size_t)t * (L + 1) * maxw;
                orc_mlp_forward(pol, p, x, g, h, maxw); /* U_k = pi(S_k, G) */
                const double* u = h + (size_t)L * maxw;
                for (int c = 0; c < p; ++c) xs[c] = x[c];
                for (int c = 0; c < d - p; ++c) xs[p + c] = u[c];
                double* xn = tx + (size_t)(t + 1) * p;
                for (int m = 0; m < p; ++m) {
                    double mu, v;
                    orc_perturb pt = {perturb_mode, perturb_seed, bg, (uint32_t)t};
                    orc_query_p(gp, m, xs, scratch, &mu, &v, tjm + ((size_t)t * p + m) * d,
                                tjv + ((size_t)t * p + m) * d, NULL, NULL, perturb_mode ? &pt : NULL);
                    double vh = v > ORC_VAR_FLOOR ? v : ORC_VAR_FLOOR;
                    double sig = sqrt(vh);
                    double e = eps_mode == 0 ? orc_rollout_eps(seed, bg, (uint32_t)t, m) : 0.0;
                    tsig[(size_t)t * p + m] = sig;
                    tvpos[(size_t)t * p + m] = v > ORC_VAR_FLOOR ? 1.0 : 0.0;
                    teps[(size_t)t * p + m] = e;
                    /* Eq.10: x_{k-1} + f_D, f_D ~ N(mu, var); absolute targets: f_D alone */
                    xn[m] = (gp->abs_target ? 0.0 : x[m]) + mu + sig * e;
                    if (trace_mu) trace_mu[((size_t)t * B + b) * p + m] = mu;
                    if (trace_var) trace_var[((size_t)t * B + b) * p + m] = v;
                }
                for (int c = 0; c < p; ++c)
                    if (!isfinite(xn[c])) dead = 1;
                if (dead) {
#pragma omp critical
                    {
                        int code = 1 + t * B + b;
                        if (bad == 0 || code < bad) bad = code;
                    }
                    break;
                }
                G += orc_reward_fn(rw, p, xn, g); /* G += r(S_{k+1}, G) */
                if (trace_x)
                    for (int c = 0; c < p; ++c) trace_x[((size_t)(t + 1) * B + b) * p + c] = xn[c];
            }
            ret[b] = G;
            if (!want_grad || dead) continue;

            /* ---------------- reverse mode (Appendix B) ---------------- */
            double* gb = gper + (size_t)b * n_theta;
            {
                const double* xT = tx + (size_t)T * p;
                double r = orc_reward_fn(rw, p, xT, g);
                for (int c = 0; c < p; ++c)
                    xbar[c] = invB * r * rw->Q[c] * (xT[c] - g[c]) / (rw->sigma_r * rw->sigma_r);
            }
            for (int t = T - 1; t >= 0; --t) {
                const double* x = tx + (size_t)t * p;
                const double* h = th + (size_t)t * (L + 1) * maxw;
                /* xs_bar = sum_m xbar_m (Jmu_m + [v>floor] eps/(2 sigma) Jv_m) */
                for (int c = 0; c < d; ++c) xsbar[c] = 0.0;
                for (int m = 0; m < p; ++m) {
                    const double* jm = tjm + ((size_t)t * p + m) * d;
                    const double* jvv = tjv + ((size_t)t * p + m) * d;
                    double f = tvpos[(size_t)t * p + m] * teps[(size_t)t * p + m] /
                               (2.0 * tsig[(size_t)t * p + m]);
                    for (int c = 0; c < d; ++c) xsbar[c] += xbar[m] * (jm[c] + f * jvv[c]);
                }
                /* MLP backward with ubar = xs_bar[p:d] */
                double* dcur = hbar;          /* delta of layer l (width out) */
                double* dprev = hbar + maxw;  /* hbar of layer l-1 */
                {
                    const double* u = h + (size_t)L * maxw;
                    int q = pol->sizes[L];
                    for (int o = 0; o < q; ++o) dcur[o] = xsbar[p + o] * (1.0 - u[o] * u[o]);
                }
                size_t off_end = n_theta;
                for (int l = L - 1; l >= 0; --l) {
                    int in = pol->sizes[l], out = pol->sizes[l + 1];
                    size_t off = off_end - ((size_t)in * out + out);
                    const double* W = pol->theta + off;
                    const double* hin = h + (size_t)l * maxw;
                    for (int o = 0; o < out; ++o) {
                        for (int i = 0; i < in; ++i) gb[off + (size_t)o * in + i] += dcur[o] * hin[i];
                        gb[off + (size_t)in * out + o] += dcur[o];
                    }
                    for (int i = 0; i < in; ++i) {
                        double acc = 0.0;
                        for (int o = 0; o < out; ++o) acc += W[(size_t)o * in + i] * dcur[o];
                        dprev[i] = l > 0 ? acc * (1.0 - hin[i] * hin[i]) : acc;
                    }
                    double* tmp = dcur;
                    dcur = dprev;
                    dprev = tmp;
                    off_end = off;
                }
                /* dcur now holds h0_bar; propagate into x_t */
                double r = orc_reward_fn(rw, p, x, g);
                for (int c = 0; c < p; ++c) {
                    double hb = dcur[c];
                    if (pol->phi_mode == 1) hb -= dcur[2 * p + c];
                    /* dx_{t+1}/dx_t = I + ... for Delta targets, no identity path for absolute */
                    xbar[c] = (gp->abs_target ? 0.0 : xbar[c]) + xsbar[c] + hb +
                              invB * r * rw->Q[c] * (x[c] - g[c]) / (rw->sigma_r * rw->sigma_r);
                }
            }
        }
        free(scratch); free(tx); free(th); free(tjm); free(tjv); free(tsig); free(tvpos);
        free(teps); free(xs); free(hbar); free(xbar); free(xsbar);
    }

    /* fixed-order reductions over trajectories */
    double cost = 0.0;
    for (int b = 0; b < B; ++b) cost += ret[b];
    *cost_out = -invB * cost;
    if (ret_out) memcpy(ret_out, ret, sizeof(double) * B);
    if (want_grad) {
        for (size_t i = 0; i < n_theta; ++i) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b) acc += gper[(size_t)b * n_theta + i];
            grad_out[i] = acc;
        }
        free(gper);
    }
    free(ret);
    return bad;
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ */
/* Algorithm 1 around the hot path            */
/* ------------------------------------------------------------------ */

/* "Sample batch of initial states S_0" (Alg.1) and goals "sampled
 * according to a distribution", uniform within the data bounds
 * (P:180): out[b][m] = lo[m] + (hi[m] - lo[m]) u with u the 23-bit uniform of
 * Philox4x32-10(key = seed, ctr = (traj_offset + b, 0, m >> 2, 2 + which))[m & 3]
 * (which = 0: S_0, 1: G).  Counter convention: DESIGN.md "Philox". */
void orc_sample_states(uint64_t seed, long long traj_offset, int B, int p, int which,
                       const double* lo, const double* hi, double* out)
{
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    for (int b = 0; b < B; ++b) {
        for (int m = 0; m < p; ++m) {
            uint32_t ctr[4] = {(uint32_t)(traj_offset + b), 0u, (uint32_t)(m >> 2), 2u + (uint32_t)which};
            uint32_t o[4];
            orc_philox4x32_10(ctr, key, o);
            double u = orc_uniform(o[m & 3]);
            out[(size_t)b * p + m] = lo[m] + (hi[m] - lo[m]) * u;
        }
    }
}

/* Adam (Kingma & Ba 2015, Algorithm 1; "for which we will use Adam", P:144;
 * SPEC S:399-403), bias-corrected, step t >= 1:
 *   m1 <- b1 m1 + (1 - b1) g;  m2 <- b2 m2 + (1 - b2) g^2
 *   m1hat = m1 / (1 - b1^t);   m2hat = m2 / (1 - b2^t)
 *   theta <- theta - lr m1hat / (sqrt(m2hat) + eps)
 * Returns 1 (and changes nothing) if any gradient entry is non-finite. */
int orc_adam_step(double* theta, const double* g, double* m1, double* m2, int n, long long t,
                  double lr, double b1, double b2, double eps)
{
    for (int i = 0; i < n; ++i)
        if (!isfinite(g[i])) return 1;
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    for (int i = 0; i < n; ++i) {
        m1[i] = b1 * m1[i] + (1.0 - b1) * g[i];
        m2[i] = b2 * m2[i] + (1.0 - b2) * g[i] * g[i];
        double m1hat = m1[i] / bc1;
        double m2hat = m2[i] / bc2;
        theta[i] -= lr * m1hat / (sqrt(m2hat) + eps);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* GP hyperparameter learning                 */
/* ------------------------------------------------------------------ */

/* Exact log marginal likelihood of one output GP and its gradient in the
 * log-hyperparameters phi = [log l_1..log l_d, log s, log sigma_n^2]
 * ("learned by maximizing the log marginal likelihood", Eq.5-6, P:77-80;
 * Eq.5 is stated up to a factor 2 and a constant and Eq.6 is garbled, so the
 * oracle writes out the standard definitions, reading R33):
 *   log p(y|X,phi) = -1/2 y^T Khat^-1 y - 1/2 log|Khat| - N/2 log(2 pi)
 *   d/dphi_j       =  1/2 y^T Khat^-1 (dKhat/dphi_j) Khat^-1 y
 *                   - 1/2 tr(Khat^-1 dKhat/dphi_j)
 *   dKhat_ij/dlog l_c = K_ij (x_ic - x_jc)^2 / l_c^2,  dKhat/dlog s = K,
 *   dKhat/dlog sigma_n^2 = sigma_n^2 I.
 * Plain steps: dense Khat, Cholesky, alpha by two triangular solves, log|Khat|
 * = 2 sum log L_ii, Khat^-1 column by column (solves against unit vectors),
 * then each derivative matrix built and contracted in full.  grad may be NULL.
 * Returns 0, or pivot + 1 if Khat is not SPD. */
int orc_mll(const double* X, int N, int d, const double* y, const double* log_hyp, double* mll,
            double* grad)
{
    double ell[16];
    for (int c = 0; c < d; ++c) ell[c] = exp(log_hyp[c]);
    double s = exp(log_hyp[d]), sn2 = exp(log_hyp[d + 1]);
    double* L = orc_khat(X, N, d, ell, s, sn2);
    if (!L) return -1;
    int rc = orc_cholesky(L, N);
    if (rc != 0) {
        free(L);
        return rc;
    }
    double* tmp = (double*)malloc(sizeof(double) * N);
    double* alpha = (double*)malloc(sizeof(double) * N);
    orc_forward_solve(L, N, y, tmp);
    orc_backward_solve_T(L, N, tmp, alpha);
    double yKy = 0.0, logdet = 0.0;
    for (int i = 0; i < N; ++i) yKy += y[i] * alpha[i];
    for (int i = 0; i < N; ++i) logdet += 2.0 * log(L[(size_t)i * N + i]);
    *mll = -0.5 * yKy - 0.5 * logdet - 0.5 * N * log(2.0 * 3.14159265358979323846);
    if (grad) {
        /* Khat^-1, column j = Khat^-1 e_j */
        double* Kinv = (double*)malloc(sizeof(double) * (size_t)N * N);
        double* e = (double*)calloc((size_t)N, sizeof(double));
        double* col = (double*)malloc(sizeof(double) * N);
        for (int j = 0; j < N; ++j) {
            e[j] = 1.0;
            orc_forward_solve(L, N, e, tmp);
            orc_backward_solve_T(L, N, tmp, col);
            e[j] = 0.0;
            for (int i = 0; i < N; ++i) Kinv[(size_t)i * N + j] = col[i];
        }
        double* D = (double*)malloc(sizeof(double) * (size_t)N * N);
        for (int jp = 0; jp < d + 2; ++jp) {
            /* D = dKhat / dphi_jp */
            for (int i = 0; i < N; ++i)
                for (int j = 0; j < N; ++j) {
                    double v;
                    if (jp < d) {
                        double diff = X[(size_t)i * d + jp] - X[(size_t)j * d + jp];
                        v = orc_kernel(X + (size_t)i * d, X + (size_t)j * d, d, ell, s) * diff * diff /
                            (ell[jp] * ell[jp]);
                    } else if (jp == d) {
                        v = orc_kernel(X + (size_t)i * d, X + (size_t)j * d, d, ell, s);
                    } else {
                        v = (i == j) ? sn2 : 0.0;
                    }
                    D[(size_t)i * N + j] = v;
                }
            /* 1/2 alpha^T D alpha - 1/2 tr(Kinv D) */
            double quad = 0.0, tr = 0.0;
            for (int i = 0; i < N; ++i) {
                double Da = 0.0;
                for (int j = 0; j < N; ++j) Da += D[(size_t)i * N + j] * alpha[j];
                quad += alpha[i] * Da;
            }
            for (int i = 0; i < N; ++i)
                for (int j = 0; j < N; ++j) tr += Kinv[(size_t)i * N + j] * D[(size_t)j * N + i];
            grad[jp] = 0.5 * quad - 0.5 * tr;
        }
        free(D);
        free(col);
        free(e);
        free(Kinv);
    }
    free(alpha);
    free(tmp);
    free(L);
    return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-1 at large N: the BBMM estimate of Eq.5-6 (P:77-81 defers to   */
/* GPyTorch [gardner2018]; reading R39).  Probes z_1..z_t are Rademacher  */
/* from Philox (key = seed, ctr = (i, n >> 2, 0x4242424D, 4), the sign   */
/* bit of word n & 3).  One batched conjugate-gradient run of exactly J  */
/* iterations (no preconditioner) solves Khat [u_0 .. u_t] = [y z_1 ..   */
/* z_t]; every probe's CG coefficients give its Lanczos tridiagonal T_i, */
/* and                                                                    */
/*   log|Khat| ~ (1/t) sum_i ||z_i||^2 e_1^T log(T_i) e_1    (SLQ)        */
/*   y^T Khat^-1 y ~ y^T u_0                                              */
/*   tr(Khat^-1 dK) ~ (1/t) sum_i u_i^T dK z_i              (Hutchinson)  */
/*   mll = -1/2 y^T u_0 - 1/2 log|Khat| - N/2 log 2 pi,                   */
/*   d mll / d phi_j = 1/2 u_0^T dK_j u_0 - 1/2 tr(Khat^-1 dK_j).         */
/* A column whose residual reaches exactly 0 stops early (its T is the   */
/* iterations done).  The eigen-decomposition of T_i is cyclic Jacobi.   */
/* ------------------------------------------------------------------ */
double orc_bbmm_probe(uint64_t seed, int i, int n)
{
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(n >> 2), 0x4242424Du, 4u};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return (o[n & 3] >> 31) ? -1.0 : 1.0;
}

/* e_1^T log(T) e_1 of a symmetric tridiagonal (diag a[0..J-1], off b[0..J-2]) by cyclic Jacobi on the
 * dense J x J matrix */
static double orc_tridiag_e1_log_e1(const double* a, const double* b, int J)
{
    double* A = (double*)calloc((size_t)J * J, sizeof(double));
    double* V = (double*)calloc((size_t)J * J, sizeof(double));
    for (int i = 0; i < J; ++i) {
        A[(size_t)i * J + i] = a[i];
        V[(size_t)i * J + i] = 1.0;
        if (i + 1 < J) A[(size_t)i * J + i + 1] = A[(size_t)(i + 1) * J + i] = b[i];
    }
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int p = 0; p < J; ++p)
            for (int q = 0; q < J; ++q) {
                if (p == q) diag += A[(size_t)p * J + p] * A[(size_t)p * J + p];
                else off += A[(size_t)p * J + q] * A[(size_t)p * J + q];
            }
        if (off <= 1e-30 * diag) break;
        for (int p = 0; p < J - 1; ++p)
            for (int q = p + 1; q < J; ++q) {
                double apq = A[(size_t)p * J + q];
                if (fabs(apq) < 1e-300) continue;
                double app = A[(size_t)p * J + p], aqq = A[(size_t)q * J + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < J; ++k) { /* A <- A J (columns p, q) */
                    double akp = A[(size_t)k * J + p], akq = A[(size_t)k * J + q];
                    A[(size_t)k * J + p] = c * akp - sn * akq;
                    A[(size_t)k * J + q] = sn * akp + c * akq;
                }
                for (int k = 0; k < J; ++k) { /* A <- J^T A (rows p, q) */
                    double apk = A[(size_t)p * J + k], aqk = A[(size_t)q * J + k];
                    A[(size_t)p * J + k] = c * apk - sn * aqk;
                    A[(size_t)q * J + k] = sn * apk + c * aqk;
                }
                for (int k = 0; k < J; ++k) { /* V <- V J */
                    double vkp = V[(size_t)k * J + p], vkq = V[(size_t)k * J + q];
                    V[(size_t)k * J + p] = c * vkp - sn * vkq;
                    V[(size_t)k * J + q] = sn * vkp + c * vkq;
                }
            }
    }
    double r = 0.0;
    for (int k = 0; k < J; ++k) r += V[k] * V[k] * log(A[(size_t)k * J + k]); /* V[0][k]^2 log lambda_k */
    free(A);
    free(V);
    return r;
}

int orc_mll_bbmm(const double* X, int N, int d, const double* y, const double* log_hyp, int t, int J,
                 uint64_t seed, double* mll, double* grad, double* logdet_out, double* quad_out)
{
    double ell[16];
    for (int c = 0; c < d; ++c) ell[c] = exp(log_hyp[c]);
    double s = exp(log_hyp[d]), sn2 = exp(log_hyp[d + 1]);
    double* K = orc_khat(X, N, d, ell, s, sn2);
    if (!K) return -1;
    const int nc = t + 1;
    double* Z = (double*)malloc(sizeof(double) * (size_t)nc * N); /* rhs columns: y, z_1..z_t */
    double* U = (double*)calloc((size_t)nc * N, sizeof(double));
    double* Rr = (double*)malloc(sizeof(double) * (size_t)nc * N);
    double* P = (double*)malloc(sizeof(double) * (size_t)nc * N);
    double* Q = (double*)malloc(sizeof(double) * (size_t)N);
    double* al = (double*)malloc(sizeof(double) * (size_t)nc * J);
    double* be = (double*)malloc(sizeof(double) * (size_t)nc * J);
    int* its = (int*)malloc(sizeof(int) * nc);
    for (int n = 0; n < N; ++n) Z[n] = y[n];
    for (int i = 1; i <= t; ++i)
        for (int n = 0; n < N; ++n) Z[(size_t)i * N + n] = orc_bbmm_probe(seed, i - 1, n);
    for (int c = 0; c < nc; ++c) {
        const double* b = Z + (size_t)c * N;
        double *u = U + (size_t)c * N, *r = Rr + (size_t)c * N, *p = P + (size_t)c * N;
        double rr = 0.0;
        for (int n = 0; n < N; ++n) {
            r[n] = b[n];
            p[n] = b[n];
            rr += b[n] * b[n];
        }
        its[c] = 0;
        for (int j = 0; j < J && rr > 0.0; ++j) {
#pragma omp parallel for schedule(static)
            for (int a = 0; a < N; ++a) {
                double acc = 0.0;
                for (int n = 0; n < N; ++n) acc += K[(size_t)a * N + n] * p[n];
                Q[a] = acc;
            }
            double pq = 0.0;
            for (int n = 0; n < N; ++n) pq += p[n] * Q[n];
            const double alpha = rr / pq;
            double rr2 = 0.0;
            for (int n = 0; n < N; ++n) {
                u[n] += alpha * p[n];
                r[n] -= alpha * Q[n];
                rr2 += r[n] * r[n];
            }
            const double beta = rr2 / rr;
            for (int n = 0; n < N; ++n) p[n] = r[n] + beta * p[n];
            al[(size_t)c * J + j] = alpha;
            be[(size_t)c * J + j] = beta;
            rr = rr2;
            its[c] = j + 1;
        }
    }
    /* SLQ over the probes */
    double logdet = 0.0;
    double* ta = (double*)malloc(sizeof(double) * J);
    double* tb = (double*)malloc(sizeof(double) * J);
    for (int i = 1; i <= t; ++i) {
        const int n = its[i];
        const double* a_ = al + (size_t)i * J;
        const double* b_ = be + (size_t)i * J;
        for (int j = 0; j < n; ++j) {
            ta[j] = 1.0 / a_[j] + (j > 0 ? b_[j - 1] / a_[j - 1] : 0.0);
            if (j + 1 < n) tb[j] = sqrt(b_[j]) / a_[j];
        }
        double zz = 0.0;
        for (int m = 0; m < N; ++m) zz += Z[(size_t)i * N + m] * Z[(size_t)i * N + m];
        logdet += zz * orc_tridiag_e1_log_e1(ta, tb, n);
    }
    logdet /= (double)t;
    double quad = 0.0;
    for (int n = 0; n < N; ++n) quad += y[n] * U[n];
    *mll = -0.5 * quad - 0.5 * logdet - 0.5 * N * log(2.0 * 3.14159265358979323846);
    if (logdet_out) *logdet_out = logdet;
    if (quad_out) *quad_out = quad;
    if (grad) {
        for (int jp = 0; jp < d + 2; ++jp) {
            /* w^T dK_jp v for (w, v) = (u_0, u_0) and (u_i, z_i) */
            double q0 = 0.0, tr = 0.0;
            for (int c = 0; c < nc; ++c) {
                const double* w = U + (size_t)c * N;
                const double* v = c == 0 ? U : Z + (size_t)c * N;
                /* per-row terms in parallel, summed in row order (thread-count independent) */
#pragma omp parallel for schedule(static)
                for (int a = 0; a < N; ++a) {
                    double row = 0.0;
                    for (int b2 = 0; b2 < N; ++b2) {
                        double dk;
                        if (jp < d) {
                            double diff = X[(size_t)a * d + jp] - X[(size_t)b2 * d + jp];
                            dk = orc_kernel(X + (size_t)a * d, X + (size_t)b2 * d, d, ell, s) * diff * diff /
                                 (ell[jp] * ell[jp]);
                        } else if (jp == d) {
                            dk = orc_kernel(X + (size_t)a * d, X + (size_t)b2 * d, d, ell, s);
                        } else {
                            dk = (a == b2) ? sn2 : 0.0;
                        }
                        row += dk * v[b2];
                    }
                    Q[a] = w[a] * row;
                }
                double acc = 0.0;
                for (int a = 0; a < N; ++a) acc += Q[a];
                if (c == 0) q0 = acc;
                else tr += acc;
            }
            grad[jp] = 0.5 * q0 - 0.5 * tr / (double)t;
        }
    }
    free(ta); free(tb); free(its); free(be); free(al); free(Q); free(P); free(Rr); free(U); free(Z); free(K);
    return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-1 at large N with GPyTorch's preconditioner (reading R40):     */
/* BBMM with a rank-k pivoted-Cholesky preconditioner [gardner2018],    */
/*   K_f ~ L L^T (k greedy pivots of the noise-free kernel matrix:     */
/*     d_n = K_f[n][n]; per step m: pivot pi = argmax over the unpivoted */
/*     n of d_n (lowest index on ties); L[n][m] = (K_f[n][pi] -          */
/*     sum_{j<m} L[n][j] L[pi][j]) / sqrt(d_pi); d_n -= L[n][m]^2;       */
/*     stop early once max d_n <= 0),                                    */
/*   P = L L^T + sn2 I, applied as P^-1 v = (v - L C^-1 L^T v) / sn2,     */
/*   C = sn2 I_k + L^T L (Woodbury), log|P| = log|C| + (N - k) log sn2;  */
/* probes z_i = L g_i[0..k) + sqrt(sn2) g_i[k..k+N) ~ N(0, P), g from     */
/* Philox (key = seed, ctr = (i, j >> 2, 0x4242424E, 5), Box-Muller word  */
/* j & 3, fp64); preconditioned CG (exactly J iterations; a column stops  */
/* once r^T P^-1 r is exactly 0) on [y z_1 .. z_t]; each probe's PCG      */
/* coefficients give the Lanczos tridiagonal T_i of P^-1/2 Khat P^-1/2,   */
/*   log|Khat| ~ log|P| + (1/t) sum_i (z_i^T P^-1 z_i) e1^T log(T_i) e1,  */
/*   tr(Khat^-1 dK) ~ (1/t) sum_i u_i^T dK (P^-1 z_i),                    */
/* quadratic term y^T u_0.  k = 0 is orc_mll_bbmm exactly.              */
/* ------------------------------------------------------------------ */
double orc_bbmm_gauss(uint64_t seed, int i, int j)
{
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(j >> 2), 0x4242424Eu, 5u};
    uint32_t o[4];
    double e[4];
    orc_philox4x32_10(ctr, key, o);
    orc_box_muller4(o, e);
    return e[j & 3];
}

/* rank-k pivoted Cholesky of K_f (row-major N x N); L is N x k row-major (L[n*k + m]); returns the
 * rank reached (<= k) */
int orc_pivoted_cholesky(const double* Kf, int N, int k, double* L, int* piv)
{
    double* dg = (double*)malloc(sizeof(double) * N);
    char* used = (char*)calloc(N, 1);
    for (int n = 0; n < N; ++n) dg[n] = Kf[(size_t)n * N + n];
    memset(L, 0, sizeof(double) * (size_t)N * k);
    int m = 0;
    for (; m < k; ++m) {
        int p = -1;
        for (int n = 0; n < N; ++n)
            if (!used[n] && (p < 0 || dg[n] > dg[p])) p = n;
        if (p < 0 || !(dg[p] > 0.0)) break;
        used[p] = 1;
        piv[m] = p;
        const double sq = sqrt(dg[p]);
        for (int n = 0; n < N; ++n) {
            double v = Kf[(size_t)n * N + p];
            for (int j = 0; j < m; ++j) v -= L[(size_t)n * k + j] * L[(size_t)p * k + j];
            L[(size_t)n * k + m] = v / sq;
        }
        for (int n = 0; n < N; ++n) dg[n] -= L[(size_t)n * k + m] * L[(size_t)n * k + m];
    }
    free(dg);
    free(used);
    return m;
}

/* in-place Cholesky of a k x k SPD matrix (lower), returns 0 or pivot+1 */
static int orc_chol_small(double* A, int k)
{
    for (int j = 0; j < k; ++j) {
        double s = A[(size_t)j * k + j];
        for (int m = 0; m < j; ++m) s -= A[(size_t)j * k + m] * A[(size_t)j * k + m];
        if (!(s > 0.0)) return j + 1;
        A[(size_t)j * k + j] = sqrt(s);
        for (int i = j + 1; i < k; ++i) {
            double v = A[(size_t)i * k + j];
            for (int m = 0; m < j; ++m) v -= A[(size_t)i * k + m] * A[(size_t)j * k + m];
            A[(size_t)i * k + j] = v / A[(size_t)j * k + j];
        }
    }
    return 0;
}

/* w = P^-1 v = (v - L C^-1 L^T v) / sn2 with C = R R^T (R lower, k x k) */
static void orc_precond_apply(const double* L, const double* R, int N, int k, double sn2, const double* v, double* w,
                              double* tmp)
{
    for (int m = 0; m < k; ++m) {
        double a = 0.0;
        for (int n = 0; n < N; ++n) a += L[(size_t)n * k + m] * v[n];
        tmp[m] = a;
    }
    for (int i = 0; i < k; ++i) { /* R x = tmp */
        double a = tmp[i];
        for (int m = 0; m < i; ++m) a -= R[(size_t)i * k + m] * tmp[m];
        tmp[i] = a / R[(size_t)i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) { /* R^T y = x */
        double a = tmp[i];
        for (int m = i + 1; m < k; ++m) a -= R[(size_t)m * k + i] * tmp[m];
        tmp[i] = a / R[(size_t)i * k + i];
    }
    for (int n = 0; n < N; ++n) {
        double a = v[n];
        for (int m = 0; m < k; ++m) a -= L[(size_t)n * k + m] * tmp[m];
        w[n] = a / sn2;
    }
}

int orc_mll_bbmm_pc(const double* X, int N, int d, const double* y, const double* log_hyp, int t, int J, int kp,
                    uint64_t seed, double* mll, double* grad, double* logdet_out, double* quad_out, int* rank_out)
{
    if (kp <= 0) {
        if (rank_out) *rank_out = 0;
        return orc_mll_bbmm(X, N, d, y, log_hyp, t, J, seed, mll, grad, logdet_out, quad_out);
    }
    double ell[16];
    for (int c = 0; c < d; ++c) ell[c] = exp(log_hyp[c]);
    double s = exp(log_hyp[d]), sn2 = exp(log_hyp[d + 1]);
    double* K = orc_khat(X, N, d, ell, s, sn2);
    if (!K) return -1;
    /* pivoted Cholesky of K_f = Khat - sn2 I */
    double* Kf = (double*)malloc(sizeof(double) * (size_t)N * N);
    memcpy(Kf, K, sizeof(double) * (size_t)N * N);
    for (int n = 0; n < N; ++n) Kf[(size_t)n * N + n] -= sn2;
    double* L0 = (double*)malloc(sizeof(double) * (size_t)N * kp);
    int* piv = (int*)malloc(sizeof(int) * kp);
    const int k = orc_pivoted_cholesky(Kf, N, kp, L0, piv);
    free(Kf);
    /* compact L to N x k, C = sn2 I + L^T L, R = chol(C), log|P| */
    double* L = (double*)malloc(sizeof(double) * (size_t)N * (k > 0 ? k : 1));
    for (int n = 0; n < N; ++n)
        for (int m = 0; m < k; ++m) L[(size_t)n * k + m] = L0[(size_t)n * kp + m];
    free(L0);
    double* R = (double*)calloc((size_t)(k > 0 ? k * k : 1), sizeof(double));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            double a = (i == j) ? sn2 : 0.0;
            for (int n = 0; n < N; ++n) a += L[(size_t)n * k + i] * L[(size_t)n * k + j];
            R[(size_t)i * k + j] = a;
        }
    if (orc_chol_small(R, k) != 0) return -2;
    double logdetP = (double)(N - k) * log(sn2);
    for (int i = 0; i < k; ++i) logdetP += 2.0 * log(R[(size_t)i * k + i]);
    const int nc = t + 1;
    double* Z = (double*)malloc(sizeof(double) * (size_t)nc * N);  /* rhs: y, z_1..z_t */
    double* W0 = (double*)malloc(sizeof(double) * (size_t)nc * N); /* P^-1 rhs */
    double* U = (double*)calloc((size_t)nc * N, sizeof(double));
    double* Rr = (double*)malloc(sizeof(double) * (size_t)N);
    double* Wv = (double*)malloc(sizeof(double) * (size_t)N);
    double* Pp = (double*)malloc(sizeof(double) * (size_t)N);
    double* Q = (double*)malloc(sizeof(double) * (size_t)N);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
    double* al = (double*)malloc(sizeof(double) * (size_t)nc * J);
    double* be = (double*)malloc(sizeof(double) * (size_t)nc * J);
    double* nz = (double*)malloc(sizeof(double) * nc);
    int* its = (int*)malloc(sizeof(int) * nc);
    for (int n = 0; n < N; ++n) Z[n] = y[n];
    for (int i = 1; i <= t; ++i)
        for (int n = 0; n < N; ++n) {
            double v = sqrt(sn2) * orc_bbmm_gauss(seed, i - 1, k + n);
            for (int m = 0; m < k; ++m) v += L[(size_t)n * k + m] * orc_bbmm_gauss(seed, i - 1, m);
            Z[(size_t)i * N + n] = v;
        }
    for (int c = 0; c < nc; ++c) {
        const double* b = Z + (size_t)c * N;
        double* u = U + (size_t)c * N;
        double* w0 = W0 + (size_t)c * N;
        for (int n = 0; n < N; ++n) Rr[n] = b[n];
        orc_precond_apply(L, R, N, k, sn2, Rr, w0, tmp);
        double rz = 0.0;
        for (int n = 0; n < N; ++n) {
            Pp[n] = w0[n];
            rz += Rr[n] * w0[n];
        }
        nz[c] = rz;
        its[c] = 0;
        for (int j = 0; j < J && rz > 0.0; ++j) {
#pragma omp parallel for schedule(static)
            for (int a = 0; a < N; ++a) {
                double acc = 0.0;
                for (int n = 0; n < N; ++n) acc += K[(size_t)a * N + n] * Pp[n];
                Q[a] = acc;
            }
            double pq = 0.0;
            for (int n = 0; n < N; ++n) pq += Pp[n] * Q[n];
            const double alpha = rz / pq;
            for (int n = 0; n < N; ++n) {
                u[n] += alpha * Pp[n];
                Rr[n] -= alpha * Q[n];
            }
            orc_precond_apply(L, R, N, k, sn2, Rr, Wv, tmp);
            double rz2 = 0.0;
            for (int n = 0; n < N; ++n) rz2 += Rr[n] * Wv[n];
            const double beta = rz2 / rz;
            for (int n = 0; n < N; ++n) Pp[n] = Wv[n] + beta * Pp[n];
            al[(size_t)c * J + j] = alpha;
            be[(size_t)c * J + j] = beta;
            rz = rz2;
            its[c] = j + 1;
        }
    }
    double logdet = 0.0;
    double* ta = (double*)malloc(sizeof(double) * J);
    double* tb = (double*)malloc(sizeof(double) * J);
    for (int i = 1; i <= t; ++i) {
        const int n = its[i];
        const double* a_ = al + (size_t)i * J;
        const double* b_ = be + (size_t)i * J;
        for (int j = 0; j < n; ++j) {
            ta[j] = 1.0 / a_[j] + (j > 0 ? b_[j - 1] / a_[j - 1] : 0.0);
            if (j + 1 < n) tb[j] = sqrt(b_[j]) / a_[j];
        }
        logdet += nz[i] * orc_tridiag_e1_log_e1(ta, tb, n);
    }
    logdet = logdetP + logdet / (double)t;
    double quad = 0.0;
    for (int n = 0; n < N; ++n) quad += y[n] * U[n];
    *mll = -0.5 * quad - 0.5 * logdet - 0.5 * N * log(2.0 * 3.14159265358979323846);
    if (logdet_out) *logdet_out = logdet;
    if (quad_out) *quad_out = quad;
    if (rank_out) *rank_out = k;
    if (grad) {
        for (int jp = 0; jp < d + 2; ++jp) {
            /* w^T dK_jp v for (w, v) = (u_0, u_0) and (u_i, P^-1 z_i) */
            double q0 = 0.0, tr = 0.0;
            for (int c = 0; c < nc; ++c) {
                const double* w = U + (size_t)c * N;
                const double* v = c == 0 ? U : W0 + (size_t)c * N;
#pragma omp parallel for schedule(static)
                for (int a = 0; a < N; ++a) {
                    double row = 0.0;
                    for (int b2 = 0; b2 < N; ++b2) {
                        double dk;
                        if (jp < d) {
                            double diff = X[(size_t)a * d + jp] - X[(size_t)b2 * d + jp];
                            dk = orc_kernel(X + (size_t)a * d, X + (size_t)b2 * d, d, ell, s) * diff * diff /
                                 (ell[jp] * ell[jp]);
                        } else if (jp == d) {
                            dk = orc_kernel(X + (size_t)a * d, X + (size_t)b2 * d, d, ell, s);
                        } else {
                            dk = (a == b2) ? sn2 : 0.0;
                        }
                        row += dk * v[b2];
                    }
                    Q[a] = w[a] * row;
                }
                double acc = 0.0;
                for (int a = 0; a < N; ++a) acc += Q[a];
                if (c == 0) q0 = acc;
                else tr += acc;
            }
            grad[jp] = 0.5 * q0 - 0.5 * tr / (double)t;
        }
    }
    free(ta); free(tb); free(its); free(nz); free(be); free(al); free(tmp); free(Q); free(Pp); free(Wv); free(Rr);
    free(U); free(W0); free(Z); free(R); free(L); free(piv); free(K);
    return 0;
}
