/*
 * TEST INFRASTRUCTURE — oracle only (never linked into the product path).
 *
 * A CPU implementation of the nine FFTW3 double-precision entry points the
 * reference's FFT layer binds (reference: proj/src/fft_plan.cpp:35,59-66,
 * 72-75,87,94; declared in oracle/include/fftw3.h).  FFTW is a third-party
 * dependency of the reference that is absent from this image and whose
 * version the reference never pins (proj/CMakeLists.txt:14-16), so the
 * reference is built against this shim to serve as the parity oracle and the
 * CPU baseline.  Algorithm (FFTW's published contract, restated):
 *
 *   r2c: row-major n[0..r-1] real -> n[0..r-2] x (n[r-1]/2+1) complex,
 *        X[k] = sum_x x[n] exp(-2 pi i <k,n>/N), unnormalised.
 *   c2r: the inverse (sign +1), unnormalised, reading only the Hermitian half;
 *        the imaginary parts of the DC and (even-length) Nyquist bins of the
 *        last axis are ignored, as FFTW's c2r does.
 *
 * Lines are transformed with a double-precision Stockham auto-sort FFT
 * (radices 4, 2, 3, 5 and a direct DFT for any other prime factor), twiddles
 * evaluated with cos/sin in double.  Two real rows are packed into one
 * complex line for the last axis.  fftw_plan_with_nthreads(n) splits the line
 * batch over n pthreads per execute (the reference's "accelerated" backend).
 */
#include "fftw3.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cpx;

#define MAX_STAGES 48
#define MAX_RANK 8
#define TWO_PI 6.283185307179586476925286766559

typedef struct {
  int n;
  int nst;
  int rad[MAX_STAGES];
  int ns[MAX_STAGES];    /* product of radices before this stage */
  cpx* tw[MAX_STAGES];   /* (R-1)*Ns twiddles exp(-2 pi i r k/(Ns R)) */
  cpx* root[MAX_STAGES]; /* R roots exp(-2 pi i q/R) for generic radices */
} line_plan;

static int g_threads = 1;

static void line_plan_init(line_plan* p, int n) {
  memset(p, 0, sizeof(*p));
  p->n = n;
  int m = n, ns = 1;
  while (m > 1) {
    int r;
    if (m % 4 == 0) r = 4;
    else if (m % 2 == 0) r = 2;
    else if (m % 3 == 0) r = 3;
    else if (m % 5 == 0) r = 5;
    else {
      r = 7;
      while (m % r != 0) r += 2;
    }
    int s = p->nst++;
    p->rad[s] = r;
    p->ns[s] = ns;
    p->tw[s] = (cpx*)malloc(sizeof(cpx) * (size_t)(r - 1) * ns + sizeof(cpx));
    for (int q = 1; q < r; ++q)
      for (int k = 0; k < ns; ++k) {
        double a = -TWO_PI * (double)q * (double)k / ((double)ns * r);
        p->tw[s][(q - 1) * ns + k].re = cos(a);
        p->tw[s][(q - 1) * ns + k].im = sin(a);
      }
    p->root[s] = (cpx*)malloc(sizeof(cpx) * r);
    for (int q = 0; q < r; ++q) {
      double a = -TWO_PI * (double)q / r;
      p->root[s][q].re = cos(a);
      p->root[s][q].im = sin(a);
    }
    ns *= r;
    m /= r;
  }
}

static void line_plan_free(line_plan* p) {
  for (int s = 0; s < p->nst; ++s) {
    free(p->tw[s]);
    free(p->root[s]);
  }
}

static inline cpx cmul(cpx a, cpx b) {
  cpx c = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return c;
}
static inline cpx cmulc(cpx a, cpx b) { /* a * conj(b) */
  cpx c = {a.re * b.re + a.im * b.im, a.im * b.re - a.re * b.im};
  return c;
}

/* In-place (result in x) transform of one contiguous line; work has n
 * entries.  sign -1 forward, +1 backward (unnormalised). */
static void line_fft(const line_plan* p, cpx* x, cpx* work, int sign) {
  const int n = p->n;
  cpx* src = x;
  cpx* dst = work;
  cpx v[64], w[64];
  for (int s = 0; s < p->nst; ++s) {
    const int R = p->rad[s], Ns = p->ns[s], m = n / R;
    const cpx* tw = p->tw[s];
    for (int j = 0; j < m; ++j) {
      const int k = j % Ns;
      const int base = (j / Ns) * Ns * R + k;
      v[0] = src[j];
      for (int r = 1; r < R; ++r) {
        cpx t = tw[(r - 1) * Ns + k];
        v[r] = sign < 0 ? cmul(src[j + r * m], t) : cmulc(src[j + r * m], t);
      }
      if (R == 2) {
        dst[base].re = v[0].re + v[1].re;
        dst[base].im = v[0].im + v[1].im;
        dst[base + Ns].re = v[0].re - v[1].re;
        dst[base + Ns].im = v[0].im - v[1].im;
      } else if (R == 4) {
        cpx a0 = {v[0].re + v[2].re, v[0].im + v[2].im};
        cpx a1 = {v[0].re - v[2].re, v[0].im - v[2].im};
        cpx a2 = {v[1].re + v[3].re, v[1].im + v[3].im};
        cpx a3 = {v[1].re - v[3].re, v[1].im - v[3].im};
        /* multiply a3 by -i (forward) or +i (backward) */
        cpx b3 = sign < 0 ? (cpx){a3.im, -a3.re} : (cpx){-a3.im, a3.re};
        dst[base].re = a0.re + a2.re;
        dst[base].im = a0.im + a2.im;
        dst[base + Ns].re = a1.re + b3.re;
        dst[base + Ns].im = a1.im + b3.im;
        dst[base + 2 * Ns].re = a0.re - a2.re;
        dst[base + 2 * Ns].im = a0.im - a2.im;
        dst[base + 3 * Ns].re = a1.re - b3.re;
        dst[base + 3 * Ns].im = a1.im - b3.im;
      } else if (R == 3) {
        const double c = -0.5, sn = (sign < 0 ? -1.0 : 1.0) * 0.86602540378443864676;
        cpx a = {v[1].re + v[2].re, v[1].im + v[2].im};
        cpx b = {v[1].re - v[2].re, v[1].im - v[2].im};
        cpx t = {v[0].re + c * a.re, v[0].im + c * a.im};
        /* i*sn*b */
        cpx u = {-sn * b.im, sn * b.re};
        dst[base].re = v[0].re + a.re;
        dst[base].im = v[0].im + a.im;
        dst[base + Ns].re = t.re + u.re;
        dst[base + Ns].im = t.im + u.im;
        dst[base + 2 * Ns].re = t.re - u.re;
        dst[base + 2 * Ns].im = t.im - u.im;
      } else if (R == 5) {
        const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
        const double sg = sign < 0 ? -1.0 : 1.0;
        const double s1 = sg * 0.95105651629515357212, s2 = sg * 0.58778525229247312917;
        cpx a1 = {v[1].re + v[4].re, v[1].im + v[4].im}, b1 = {v[1].re - v[4].re, v[1].im - v[4].im};
        cpx a2 = {v[2].re + v[3].re, v[2].im + v[3].im}, b2 = {v[2].re - v[3].re, v[2].im - v[3].im};
        cpx t1 = {v[0].re + c1 * a1.re + c2 * a2.re, v[0].im + c1 * a1.im + c2 * a2.im};
        cpx t2 = {v[0].re + c2 * a1.re + c1 * a2.re, v[0].im + c2 * a1.im + c1 * a2.im};
        /* u = i*(s1 b1 + s2 b2), w = i*(s2 b1 - s1 b2) */
        cpx u = {-(s1 * b1.im + s2 * b2.im), s1 * b1.re + s2 * b2.re};
        cpx w = {-(s2 * b1.im - s1 * b2.im), s2 * b1.re - s1 * b2.re};
        dst[base].re = v[0].re + a1.re + a2.re;
        dst[base].im = v[0].im + a1.im + a2.im;
        dst[base + Ns].re = t1.re + u.re;
        dst[base + Ns].im = t1.im + u.im;
        dst[base + 4 * Ns].re = t1.re - u.re;
        dst[base + 4 * Ns].im = t1.im - u.im;
        dst[base + 2 * Ns].re = t2.re + w.re;
        dst[base + 2 * Ns].im = t2.im + w.im;
        dst[base + 3 * Ns].re = t2.re - w.re;
        dst[base + 3 * Ns].im = t2.im - w.im;
      } else {
        const cpx* rt = p->root[s];
        for (int q = 0; q < R; ++q) {
          cpx acc = {0, 0};
          for (int r = 0; r < R; ++r) {
            cpx t = rt[(r * q) % R];
            cpx pr = sign < 0 ? cmul(v[r], t) : cmulc(v[r], t);
            acc.re += pr.re;
            acc.im += pr.im;
          }
          w[q] = acc;
        }
        for (int q = 0; q < R; ++q) dst[base + q * Ns] = w[q];
      }
    }
    cpx* t = src;
    src = dst;
    dst = t;
  }
  if (src != x) memcpy(x, src, sizeof(cpx) * (size_t)n);
}

struct fftw_plan_s {
  int c2r;
  int rank;
  int n[MAX_RANK];
  double* real;
  cpx* cplx;
  int nthreads;
  line_plan lp[MAX_RANK];
};

int fftw_init_threads(void) { return 1; }
void fftw_plan_with_nthreads(int nthreads) { g_threads = nthreads < 1 ? 1 : nthreads; }
double* fftw_alloc_real(size_t n) { return (double*)aligned_alloc(64, ((n ? n : 1) * 8 + 63) / 64 * 64); }
fftw_complex* fftw_alloc_complex(size_t n) {
  return (fftw_complex*)aligned_alloc(64, ((n ? n : 1) * 16 + 63) / 64 * 64);
}
void fftw_free(void* p) { free(p); }

static fftw_plan make_plan(int c2r, int rank, const int* n, double* real, cpx* c) {
  if (rank < 1 || rank > MAX_RANK) return NULL;
  fftw_plan p = (fftw_plan)calloc(1, sizeof(struct fftw_plan_s));
  p->c2r = c2r;
  p->rank = rank;
  for (int a = 0; a < rank; ++a) {
    if (n[a] < 1) {
      free(p);
      return NULL;
    }
    p->n[a] = n[a];
    line_plan_init(&p->lp[a], n[a]);
  }
  p->real = real;
  p->cplx = c;
  p->nthreads = g_threads;
  return p;
}

fftw_plan fftw_plan_dft_r2c(int rank, const int* n, double* in, fftw_complex* out,
                            unsigned flags) {
  (void)flags;
  return make_plan(0, rank, n, in, (cpx*)out);
}
fftw_plan fftw_plan_dft_c2r(int rank, const int* n, fftw_complex* in, double* out,
                            unsigned flags) {
  (void)flags;
  return make_plan(1, rank, n, out, (cpx*)in);
}
void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  for (int a = 0; a < p->rank; ++a) line_plan_free(&p->lp[a]);
  free(p);
}

/* ---- parallel helpers --------------------------------------------------- */

typedef struct {
  fftw_plan p;
  int phase; /* -1: last-axis pass, else axis index */
  long lo, hi;
} job;

enum { BLOCK = 16 };

/* Last axis: pairs of real rows <-> one complex line. */
static void last_axis(fftw_plan p, long lo, long hi) {
  const int nx = p->n[p->rank - 1], hx = nx / 2 + 1;
  long rows = 1;
  for (int a = 0; a < p->rank - 1; ++a) rows *= p->n[a];
  cpx* z = (cpx*)malloc(sizeof(cpx) * (size_t)nx);
  cpx* wk = (cpx*)malloc(sizeof(cpx) * (size_t)nx);
  for (long pr = lo; pr < hi; ++pr) {
    const long ra = 2 * pr, rb = 2 * pr + 1;
    const int has_b = rb < rows;
    double* xa = p->real + ra * nx;
    double* xb = has_b ? p->real + rb * nx : NULL;
    cpx* ca = p->cplx + ra * hx;
    cpx* cb = has_b ? p->cplx + rb * hx : NULL;
    if (!p->c2r) {
      for (int i = 0; i < nx; ++i) {
        z[i].re = xa[i];
        z[i].im = has_b ? xb[i] : 0.0;
      }
      line_fft(&p->lp[p->rank - 1], z, wk, -1);
      for (int k = 0; k < hx; ++k) {
        cpx zk = z[k], zn = z[(nx - k) % nx];
        ca[k].re = 0.5 * (zk.re + zn.re);
        ca[k].im = 0.5 * (zk.im - zn.im);
        if (has_b) {
          cb[k].re = 0.5 * (zk.im + zn.im);
          cb[k].im = -0.5 * (zk.re - zn.re);
        }
      }
    } else {
      for (int k = 0; k < nx; ++k) {
        cpx a, b = {0, 0};
        if (k < hx) {
          a = ca[k];
          if (has_b) b = cb[k];
          if (k == 0 || 2 * k == nx) {
            a.im = 0;
            b.im = 0;
          }
        } else {
          a = ca[nx - k];
          a.im = -a.im;
          if (has_b) {
            b = cb[nx - k];
            b.im = -b.im;
          }
        }
        z[k].re = a.re - b.im;
        z[k].im = a.im + b.re;
      }
      line_fft(&p->lp[p->rank - 1], z, wk, +1);
      for (int i = 0; i < nx; ++i) {
        xa[i] = z[i].re;
        if (has_b) xb[i] = z[i].im;
      }
    }
  }
  free(z);
  free(wk);
}

/* Complex lines along `axis` of the (n[0..r-2], hx) complex array; work items
 * are (outer, inner-block) pairs. */
static void axis_pass(fftw_plan p, int axis, long lo, long hi) {
  const int r = p->rank, nx = p->n[r - 1], hx = nx / 2 + 1;
  long inner = hx;
  for (int a = axis + 1; a < r - 1; ++a) inner *= p->n[a];
  const int len = p->n[axis];
  const long nblk = (inner + BLOCK - 1) / BLOCK;
  const int sign = p->c2r ? +1 : -1;
  cpx* buf = (cpx*)malloc(sizeof(cpx) * (size_t)len * BLOCK);
  cpx* wk = (cpx*)malloc(sizeof(cpx) * (size_t)len);
  for (long it = lo; it < hi; ++it) {
    const long outer = it / nblk, b0 = (it % nblk) * BLOCK;
    const int nb = (int)((inner - b0) < BLOCK ? (inner - b0) : BLOCK);
    cpx* base = p->cplx + outer * (long)len * inner + b0;
    for (int i = 0; i < len; ++i)
      for (int b = 0; b < nb; ++b) buf[b * len + i] = base[(long)i * inner + b];
    for (int b = 0; b < nb; ++b) line_fft(&p->lp[axis], buf + (long)b * len, wk, sign);
    for (int i = 0; i < len; ++i)
      for (int b = 0; b < nb; ++b) base[(long)i * inner + b] = buf[b * len + i];
  }
  free(buf);
  free(wk);
}

static void* run_job(void* arg) {
  job* j = (job*)arg;
  if (j->phase < 0) last_axis(j->p, j->lo, j->hi);
  else axis_pass(j->p, j->phase, j->lo, j->hi);
  return NULL;
}

static void run_phase(fftw_plan p, int phase, long items) {
  int nt = p->nthreads;
  if (nt > items) nt = (int)(items > 0 ? items : 1);
  job jobs[256];
  pthread_t th[256];
  if (nt > 256) nt = 256;
  for (int t = 0; t < nt; ++t) {
    jobs[t].p = p;
    jobs[t].phase = phase;
    jobs[t].lo = items * t / nt;
    jobs[t].hi = items * (t + 1) / nt;
  }
  if (nt == 1) {
    run_job(&jobs[0]);
    return;
  }
  for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

static long axis_items(fftw_plan p, int axis) {
  const int r = p->rank, hx = p->n[r - 1] / 2 + 1;
  long inner = hx, outer = 1;
  for (int a = axis + 1; a < r - 1; ++a) inner *= p->n[a];
  for (int a = 0; a < axis; ++a) outer *= p->n[a];
  return outer * ((inner + BLOCK - 1) / BLOCK);
}

void fftw_execute(const fftw_plan p) {
  if (!p) return;
  long rows = 1;
  for (int a = 0; a < p->rank - 1; ++a) rows *= p->n[a];
  const long pairs = (rows + 1) / 2;
  if (!p->c2r) {
    run_phase(p, -1, pairs);
    for (int a = p->rank - 2; a >= 0; --a) run_phase(p, a, axis_items(p, a));
  } else {
    for (int a = 0; a <= p->rank - 2; ++a) run_phase(p, a, axis_items(p, a));
    run_phase(p, -1, pairs);
  }
}
