/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU implementation of the Gated DeltaNet (GDN) recurrence,
 * token by token.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2605_19049_b200/) never links, imports or executes it, and this
 * file shares no code, header, table or constant with it.
 *
 * What it computes (the plain definition the KV-buffered method must reach):
 *
 *   PAPER.md:362-365 (Appendix A, eq:gated_state / eq:recurrent_gdn_decoding),
 *   paper (row-vector) convention, S in R^{d_k x d_v}:
 *       S~_{t-1} = alpha_t S_{t-1}
 *       S_t      = (I - beta_t k_t^T k_t) S~_{t-1} + beta_t k_t^T v_t
 *       o_t      = q_t S_t                     (output read-out)
 *
 *   This file stores the transpose (north-star convention, DESIGN.md reading
 *   Z1): S in R^{d_v x d_k}, row j = value index, column r = key index, so
 *       S  <- alpha_t S                                    (decay old state only, Z8)
 *       m_j = sum_r S[j][r] k_t[r]                         (ascending r, fixed order)
 *       u_j = beta_w,t v_t[j] - beta_e,t m_j               (delta value)
 *       S[j][r] += u_j k_t[r]
 *       o_t[j] = sum_r S[j][r] q_t[r]
 *
 *   GDN ties the erase and write coefficients: beta_e = beta_w = beta_t
 *   ("(I - beta k^T k) ... + beta k^T v").  Keeping them separate
 *   lets the self-tests reach vanilla linear attention (alpha = 1, beta_e = 0,
 *   beta_w = 1 gives S_t = S_{t-1} + v_t k_t^T) — DESIGN.md Z7.
 *
 * Parallelism: independent sequences (one per (request slot, V head)) are
 * split across POSIX threads.  Each sequence is processed exactly as above.
 */
#include <pthread.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int d_k, d_v, n_tok;
    const double *q, *k, *v;           /* [n_seq][n_tok][d] */
    const double *alpha, *beta_e, *beta_w; /* [n_seq][n_tok] */
    double *o;                         /* [n_seq][n_tok][d_v] or NULL */
    double *S;                         /* [n_seq][d_v][d_k], updated in place */
    int seq_begin, seq_end;
} oracle_job;

static void run_one_sequence(const oracle_job *J, int s)
{
    const int dk = J->d_k, dv = J->d_v, T = J->n_tok;
    double *S = J->S + (size_t)s * dv * dk;
    for (int t = 0; t < T; ++t) {
        const size_t tok = (size_t)s * T + t;
        const double *q = J->q + tok * dk;
        const double *k = J->k + tok * dk;
        const double *v = J->v + tok * dv;
        const double a = J->alpha[tok];
        const double be = J->beta_e[tok];
        const double bw = J->beta_w[tok];
        /* S~ = alpha S */
        for (int j = 0; j < dv; ++j)
            for (int r = 0; r < dk; ++r)
                S[(size_t)j * dk + r] *= a;
        for (int j = 0; j < dv; ++j) {
            double *row = S + (size_t)j * dk;
            double m = 0.0;
            for (int r = 0; r < dk; ++r)
                m += row[r] * k[r];
            const double u = bw * v[j] - be * m;
            for (int r = 0; r < dk; ++r)
                row[r] += u * k[r];
            if (J->o) {
                double acc = 0.0;
                for (int r = 0; r < dk; ++r)
                    acc += row[r] * q[r];
                J->o[tok * dv + j] = acc;
            }
        }
    }
}

static void *worker(void *arg)
{
    const oracle_job *J = (const oracle_job *)arg;
    for (int s = J->seq_begin; s < J->seq_end; ++s)
        run_one_sequence(J, s);
    return NULL;
}

/*
 * oracle_gdn_run: advance n_seq independent GDN sequences by n_tok tokens.
 *   S      [n_seq][d_v][d_k]  in: start state, out: state after n_tok tokens
 *   q, k   [n_seq][n_tok][d_k]; v [n_seq][n_tok][d_v]
 *   alpha, beta_e, beta_w [n_seq][n_tok]
 *   o      [n_seq][n_tok][d_v] (may be NULL)
 *   n_threads <= 0 -> 1
 * Returns 0, or -1 on invalid sizes / thread failure.
 */
int oracle_gdn_run(int n_seq, int d_k, int d_v, int n_tok,
                   double *S, const double *q, const double *k, const double *v,
                   const double *alpha, const double *beta_e, const double *beta_w,
                   double *o, int n_threads)
{
    if (n_seq < 0 || d_k <= 0 || d_v <= 0 || n_tok < 0) return -1;
    if (n_seq == 0 || n_tok == 0) return 0;
    if (n_threads <= 0) n_threads = 1;
    if (n_threads > n_seq) n_threads = n_seq;
    oracle_job *jobs = (oracle_job *)calloc((size_t)n_threads, sizeof(oracle_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    int rc = 0, started = 0;
    for (int i = 0; i < n_threads; ++i) {
        oracle_job *J = &jobs[i];
        J->d_k = d_k; J->d_v = d_v; J->n_tok = n_tok;
        J->q = q; J->k = k; J->v = v;
        J->alpha = alpha; J->beta_e = beta_e; J->beta_w = beta_w;
        J->o = o; J->S = S;
        J->seq_begin = (int)((long long)n_seq * i / n_threads);
        J->seq_end = (int)((long long)n_seq * (i + 1) / n_threads);
        if (n_threads == 1) { worker(J); continue; }
        if (pthread_create(&th[i], NULL, worker, J) != 0) { rc = -1; break; }
        ++started;
    }
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(jobs); free(th);
    return rc;
}
