/*
 * ORACLE -- test infrastructure only (never linked into librnsw.so, never
 * measured as the product).
 *
 * Plain-C restatement of the reference's exact convolution oracle
 * ``direct_conv`` (rw/layer.py:81-103): y[b,ho,wo,k] = sum over (u,v,c) of
 * xpad[b,ho+u,wo+v,c] * w[u,v,c,k], correlation, zero padding, stride 1,
 * NHWC activations and (R,R,C,K) weights.  The reference accumulates in
 * guarded int32 (rw/gemm.py:43-88); here int64 accumulation is narrowed to
 * int32, identical whenever the reference does not raise OverflowRisk.
 * pthreads over output rows keep the full-size checks (e.g. VGG16 layers)
 * within seconds.
 *
 * Also: the reference's modular sandwich and MRC as scalar loops, used by the
 * tests to check single tiles independently of numpy.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct {
  const int8_t *x, *wt;
  int B, H, W, C, K, R, pad, Ho, Wo;
  int32_t* y;
  int row0, row1; /* rows of the flattened (b, ho) range */
} conv_job;

static void* conv_rows(void* arg) {
  const conv_job* j = (const conv_job*)arg;
  for (int row = j->row0; row < j->row1; ++row) {
    const int b = row / j->Ho, ho = row % j->Ho;
    for (int wo = 0; wo < j->Wo; ++wo)
      for (int k = 0; k < j->K; ++k) {
        int64_t acc = 0;
        for (int u = 0; u < j->R; ++u) {
          const int h = ho + u - j->pad;
          if (h < 0 || h >= j->H) continue;
          for (int v = 0; v < j->R; ++v) {
            const int ww = wo + v - j->pad;
            if (ww < 0 || ww >= j->W) continue;
            const int8_t* xp = j->x + (((size_t)b * j->H + h) * j->W + ww) * j->C;
            const int8_t* wp = j->wt + (((size_t)k * j->R + u) * j->R + v) * j->C;
            int32_t s = 0;
            for (int c = 0; c < j->C; ++c) s += (int32_t)xp[c] * (int32_t)wp[c];
            acc += s;
          }
        }
        j->y[(((size_t)b * j->Ho + ho) * j->Wo + wo) * j->K + k] = (int32_t)acc;
      }
  }
  return NULL;
}

int oracle_direct_conv(const int8_t* x, const int8_t* w, int B, int H, int W, int C, int K, int R, int pad,
                       int32_t* y) {
  const int Ho = H + 2 * pad - R + 1, Wo = W + 2 * pad - R + 1;
  if (Ho < 1 || Wo < 1) return 1;
  /* transpose weights to [k][u][v][c] so the inner loop runs over contiguous c */
  int8_t* wt = (int8_t*)malloc((size_t)K * R * R * C);
  if (!wt) return 2;
  for (int u = 0; u < R; ++u)
    for (int v = 0; v < R; ++v)
      for (int c = 0; c < C; ++c)
        for (int k = 0; k < K; ++k) wt[(((size_t)k * R + u) * R + v) * C + c] = w[(((size_t)u * R + v) * C + c) * K + k];
  long ncpu = sysconf(_SC_NPROCESSORS_ONLN);
  int nt = ncpu < 1 ? 1 : (ncpu > 64 ? 64 : (int)ncpu);
  const int rows = B * Ho;
  if (nt > rows) nt = rows;
  pthread_t th[64];
  conv_job jobs[64];
  for (int t = 0; t < nt; ++t) {
    conv_job jb = {x, wt, B, H, W, C, K, R, pad, Ho, Wo, y, (int)((int64_t)rows * t / nt),
                   (int)((int64_t)rows * (t + 1) / nt)};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, conv_rows, &jobs[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(wt);
  return 0;
}

static int64_t sym64(int64_t x, int64_t m) {
  int64_t r = x % m;
  if (r < 0) r += m;
  return r > (m - 1) / 2 ? r - m : r;
}

/* out (rows_l x cols_r) = (L (rows_l x n) @ X (n x n2) mod m) @ Rt (n2 x cols_r) mod m,
 * the reference's _sandwich_mod (rw/kernel.py:21-30) for one tile. */
void oracle_sandwich_mod(const int32_t* L, const int32_t* X, const int32_t* Rm, int rows_l, int n, int n2,
                         int cols_r, int32_t m, int32_t* out) {
  int64_t* t = (int64_t*)malloc(sizeof(int64_t) * rows_l * n2);
  for (int i = 0; i < rows_l; ++i)
    for (int j = 0; j < n2; ++j) {
      int64_t s = 0;
      for (int a = 0; a < n; ++a) s += (int64_t)L[i * n + a] * X[a * n2 + j];
      t[i * n2 + j] = sym64(s, m);
    }
  for (int i = 0; i < rows_l; ++i)
    for (int j = 0; j < cols_r; ++j) {
      int64_t s = 0;
      for (int a = 0; a < n2; ++a) s += t[i * n2 + a] * Rm[a * cols_r + j];
      out[i * cols_r + j] = (int32_t)sym64(s, m);
    }
  free(t);
}

/* Mixed-radix reconstruction of one residue vector (rw/residue.py:109-127). */
int64_t oracle_mrc(const int32_t* res, const int32_t* moduli, int n) {
  int64_t d[8];
  for (int j = 0; j < n; ++j) {
    const int64_t m = moduli[j];
    int64_t t = ((int64_t)res[j] % m + m) % m;
    for (int i = 0; i < j; ++i) {
      /* inverse of moduli[i] mod m by extended Euclid */
      int64_t a = moduli[i] % m, b = m, x0 = 1, x1 = 0;
      while (b) {
        int64_t q = a / b, tmp = a - q * b;
        a = b;
        b = tmp;
        tmp = x0 - q * x1;
        x0 = x1;
        x1 = tmp;
      }
      const int64_t inv = ((x0 % m) + m) % m;
      t = (((t - d[i]) * inv) % m + m) % m;
    }
    d[j] = t;
  }
  int64_t x = d[n - 1], D = 1;
  for (int j = n - 2; j >= 0; --j) x = x * moduli[j] + d[j];
  for (int j = 0; j < n; ++j) D *= moduli[j];
  return x > (D - 1) / 2 ? x - D : x;
}
