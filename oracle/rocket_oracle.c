/*
 * rocket_oracle.c — CPU restatement of the reference ROCKET transform.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline — never as a product path.
 *
 * Follows, line by line, the arithmetic of
 *   /root/reference/pkg/src/gridrocket/engine.py:148-190   (_run_batch)
 *   /root/reference/pkg/src/gridrocket/engine.py:193-249   (_run_batch_mpv)
 *   /root/reference/pkg/src/gridrocket/reference.py:1-17   (arithmetic contract)
 * in float32 ("single") and float64 ("double"):
 *   acc = 0; for c in channels(k) ascending: for j < len: idx = t - p + j*d;
 *   if 0 <= idx < L: acc = RN(acc + RN(w*x))   -- no FMA contraction
 *   acc = RN(acc + bias); count += acc > 0; max = acc > max ? acc : max
 *   out[i, k*fpk] = (T)((double)count / (double)l_out); out[.., +1] = max
 *   mpv: ascending-position T-sum of positives, divided in double.
 * Compiled with -ffp-contract=off so gcc keeps mul and add separate (the
 * numba/LLVM reference emits vmulss + vaddss).
 *
 * Rows are independent (engine.py:157), so the row loop is split across
 * pthreads; results do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const void* x;
  int64_t n, C, L;
  const int32_t *lengths, *dilations, *paddings;
  const void *biases, *wflat;
  const int64_t *woff, *choff;
  const int32_t *chidx, *chcnt;
  int64_t K;
  int32_t fpk;
  void* out;
  int64_t ld_out;
  int64_t row_begin, row_end;
  int64_t executed;
  int dbl;
} job_t;

#define DEFINE_ROWS(T, NAME)                                                             \
  static void NAME(job_t* j) {                                                           \
    const T* x = (const T*)j->x;                                                         \
    const T* w = (const T*)j->wflat;                                                     \
    const T* b = (const T*)j->biases;                                                    \
    T* out = (T*)j->out;                                                                 \
    const int64_t L = j->L, C = j->C;                                                    \
    T* vals = NULL;                                                                      \
    int64_t vcap = 0;                                                                    \
    int64_t executed = 0;                                                                \
    for (int64_t i = j->row_begin; i < j->row_end; ++i) {                                \
      const T* xi = x + i * C * L;                                                       \
      for (int64_t k = 0; k < j->K; ++k) {                                               \
        const int64_t lk = j->lengths[k], d = j->dilations[k], p = j->paddings[k];       \
        const int64_t l_out = L + 2 * p - (lk - 1) * d;                                  \
        const int64_t nc = j->chcnt[k], wb = j->woff[k], cb = j->choff[k];               \
        if (j->fpk == 3 && l_out > vcap) {                                               \
          free(vals);                                                                    \
          vcap = l_out;                                                                  \
          vals = (T*)malloc(sizeof(T) * vcap);                                           \
        }                                                                                \
        int64_t count = 0;                                                               \
        T running_max = (T)-INFINITY;                                                    \
        for (int64_t t = 0; t < l_out; ++t) {                                            \
          T acc = (T)0;                                                                  \
          for (int64_t c = 0; c < nc; ++c) {                                             \
            const T* xc = xi + (int64_t)j->chidx[cb + c] * L;                            \
            const T* wr = w + wb + c * lk;                                               \
            for (int64_t q = 0; q < lk; ++q) {                                           \
              const int64_t idx = t - p + q * d;                                         \
              if (idx >= 0 && idx < L) {                                                 \
                T prod = wr[q] * xc[idx];                                                \
                acc = acc + prod;                                                        \
              }                                                                          \
            }                                                                            \
          }                                                                              \
          acc = acc + b[k];                                                              \
          if (acc > 0) count += 1;                                                       \
          if (acc > running_max) running_max = acc;                                      \
          if (j->fpk == 3) vals[t] = acc;                                                \
        }                                                                                \
        T* o = out + i * j->ld_out + k * j->fpk;                                         \
        o[0] = (T)((double)count / (double)l_out);                                       \
        o[1] = running_max;                                                              \
        if (j->fpk == 3) {                                                               \
          if (count > 0) {                                                               \
            T psum = (T)0;                                                               \
            for (int64_t t = 0; t < l_out; ++t)                                          \
              if (vals[t] > 0) psum = psum + vals[t];                                    \
            o[2] = (T)((double)psum / (double)count);                                    \
          } else {                                                                       \
            o[2] = (T)0;                                                                 \
          }                                                                              \
        }                                                                                \
        executed += l_out;                                                               \
      }                                                                                  \
    }                                                                                    \
    free(vals);                                                                          \
    j->executed = executed;                                                              \
  }

DEFINE_ROWS(float, rows_f32)
DEFINE_ROWS(double, rows_f64)

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  if (j->dbl)
    rows_f64(j);
  else
    rows_f32(j);
  return NULL;
}

/* Same argument order as engine._run_batch (engine.py:148-150) plus sizes.
 * dbl = 0: x/biases/wflat/out are float32; dbl = 1: float64.
 * Returns the number of executed dot-product positions. */
int64_t rko_run_batch(int dbl, const void* x, int64_t n, int64_t C, int64_t L, const int32_t* lengths,
                      const int32_t* dilations, const int32_t* paddings, const void* biases, const void* wflat,
                      const int64_t* woff, const int32_t* chidx, const int64_t* choff, const int32_t* chcnt,
                      int64_t K, int32_t fpk, void* out, int64_t ld_out, int64_t row0, int32_t nthreads) {
  if (n <= 0) return 0;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = (int32_t)n;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  const size_t esz = dbl ? sizeof(double) : sizeof(float);
  void* out0 = (char*)out + (size_t)(row0 * ld_out) * esz;
  for (int32_t t = 0; t < nthreads; ++t) {
    job_t* j = &jobs[t];
    j->x = x;
    j->n = n;
    j->C = C;
    j->L = L;
    j->lengths = lengths;
    j->dilations = dilations;
    j->paddings = paddings;
    j->biases = biases;
    j->wflat = wflat;
    j->woff = woff;
    j->chidx = chidx;
    j->choff = choff;
    j->chcnt = chcnt;
    j->K = K;
    j->fpk = fpk;
    j->out = out0;
    j->ld_out = ld_out;
    j->row_begin = n * t / nthreads;
    j->row_end = n * (t + 1) / nthreads;
    j->dbl = dbl;
  }
  for (int32_t t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  int64_t executed = jobs[0].executed;
  for (int32_t t = 1; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    executed += jobs[t].executed;
  }
  free(jobs);
  free(th);
  return executed;
}

/* Full convolution vector of one kernel in float64 (reference.py:101-139,
 * convolve(..., dtype=float64)); used to certify fast-mode PPV flips. */
void rko_convolve_f64(const double* x, int64_t L, const int32_t* chidx, int64_t nc, const double* w, int64_t lk,
                      double bias, int64_t d, int64_t p, double* out, int64_t l_out) {
  for (int64_t t = 0; t < l_out; ++t) {
    double acc = 0.0;
    for (int64_t c = 0; c < nc; ++c) {
      const double* xc = x + (int64_t)chidx[c] * L;
      for (int64_t q = 0; q < lk; ++q) {
        const int64_t idx = t - p + q * d;
        if (idx >= 0 && idx < L) {
          double prod = w[c * lk + q] * xc[idx];
          acc = acc + prod;
        }
      }
    }
    out[t] = acc + bias;
  }
}

/* Floating-point certification of single-precision cells (the fast-mode
 * tolerance, tests/parity.py).  For each requested (row, kernel) cell the
 * convolution is recomputed exactly enough in float64 from the SAME float32
 * operands the transforms use (the bank cast to float32 as engine.py:275-276
 * does; a float32 x float32 product is exact in float64), and each output t
 * gets the classical forward-error bound of a float32 evaluation in any
 * order, with or without FMA (Higham, Accuracy and Stability of Numerical
 * Algorithms, 2nd ed., eq. 3.5 / Lemma 3.1):
 *     e_t = gamma(m + 1) * (|b| + sum_taps |w * x|),
 *     gamma(n) = n u / (1 - n u),  u = 2^-24,  m = in-range taps at t.
 * Outputs per cell:
 *   max64[i]   max_t v64[t]                (the float64 MAX)
 *   maxerr[i]  max_t e_t                   (|MAX_f32 - max64| <= maxerr)
 *   near[i]    #{t : |v64[t]| < near_abs}  (the north star's 1e-6 band)
 *   unsure[i]  #{t : |v64[t]| <= max(near_abs, e_t)} (sign not decided by
 *              float32 arithmetic)
 *   pos[i]     #{t : v64[t] > 0}
 *   psum64[i]  sum of the positive v64[t]
 *   psumerr[i] sum over t with v64[t] > -e_t of 2 e_t (a bound on how far
 *              any float32 positive sum's terms and membership move it)
 */
typedef struct {
  const float* x;
  int64_t C, L;
  const int32_t *lengths, *dilations, *paddings, *chidx, *chcnt;
  const float *biases, *wflat;
  const int64_t *woff, *choff, *rows, *ks;
  double near_abs;
  double *max64, *maxerr, *psum64, *psumerr;
  int64_t *near, *unsure, *pos;
  int64_t begin, end;
} cert_t;

static void* cert_worker(void* arg) {
  cert_t* c = (cert_t*)arg;
  const double u = ldexp(1.0, -24);
  for (int64_t i = c->begin; i < c->end; ++i) {
    const int64_t k = c->ks[i];
    const float* xi = c->x + c->rows[i] * c->C * c->L;
    const int64_t L = c->L, lk = c->lengths[k], d = c->dilations[k], p = c->paddings[k];
    const int64_t l_out = L + 2 * p - (lk - 1) * d, nc = c->chcnt[k];
    const float* w = c->wflat + c->woff[k];
    const double b = (double)c->biases[k];
    double mx = -INFINITY, mxe = 0.0, ps = 0.0, pse = 0.0;
    int64_t near = 0, unsure = 0, pos = 0;
    for (int64_t t = 0; t < l_out; ++t) {
      double acc = 0.0, mag = fabs(b);
      int64_t m = 0;
      for (int64_t ch = 0; ch < nc; ++ch) {
        const float* xc = xi + (int64_t)c->chidx[c->choff[k] + ch] * L;
        for (int64_t q = 0; q < lk; ++q) {
          const int64_t idx = t - p + q * d;
          if (idx >= 0 && idx < L) {
            const double prod = (double)w[ch * lk + q] * (double)xc[idx];
            acc += prod;
            mag += fabs(prod);
            ++m;
          }
        }
      }
      const double v = acc + b;
      const double g = (double)(m + 1) * u / (1.0 - (double)(m + 1) * u);
      /* + 2^-50 mag: the float64 evaluation's own rounding */
      const double e = g * mag + ldexp(mag, -50);
      if (v > mx) mx = v;
      if (e > mxe) mxe = e;
      if (fabs(v) < c->near_abs) ++near;
      if (fabs(v) <= (e > c->near_abs ? e : c->near_abs)) ++unsure;
      if (v > 0) {
        ++pos;
        ps += v;
      }
      if (v > -e) pse += 2.0 * e;
    }
    c->max64[i] = mx;
    c->maxerr[i] = mxe;
    c->near[i] = near;
    c->unsure[i] = unsure;
    c->pos[i] = pos;
    c->psum64[i] = ps;
    c->psumerr[i] = pse;
  }
  return NULL;
}

void rko_cell_cert(const float* x, int64_t C, int64_t L, const int32_t* lengths, const int32_t* dilations,
                   const int32_t* paddings, const float* biases, const float* wflat, const int64_t* woff,
                   const int32_t* chidx, const int64_t* choff, const int32_t* chcnt, const int64_t* rows,
                   const int64_t* ks, int64_t ncells, double near_abs, double* max64, double* maxerr, int64_t* near,
                   int64_t* unsure, int64_t* pos, double* psum64, double* psumerr, int32_t nthreads) {
  if (ncells <= 0) return;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ncells) nthreads = (int32_t)ncells;
  cert_t* jobs = (cert_t*)calloc((size_t)nthreads, sizeof(cert_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int32_t t = 0; t < nthreads; ++t) {
    cert_t* j = &jobs[t];
    j->x = x;
    j->C = C;
    j->L = L;
    j->lengths = lengths;
    j->dilations = dilations;
    j->paddings = paddings;
    j->chidx = chidx;
    j->chcnt = chcnt;
    j->biases = biases;
    j->wflat = wflat;
    j->woff = woff;
    j->choff = choff;
    j->rows = rows;
    j->ks = ks;
    j->near_abs = near_abs;
    j->max64 = max64;
    j->maxerr = maxerr;
    j->psum64 = psum64;
    j->psumerr = psumerr;
    j->near = near;
    j->unsure = unsure;
    j->pos = pos;
    j->begin = ncells * t / nthreads;
    j->end = ncells * (t + 1) / nthreads;
  }
  for (int32_t t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, cert_worker, &jobs[t]);
  cert_worker(&jobs[0]);
  for (int32_t t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
}
