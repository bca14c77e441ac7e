/* capi_demo.c -- the drop-in boundary used from plain C (no Python, no torch,
 * no CUDA headers): include/clifford_b200.h + libclifford_b200.so only.
 *
 * Checks the fp32-mode conv (host-buffer entry point) against an fp64 direct
 * convolution restated here from the reference (conv.py:151-182: out[b,co,p] =
 * bias[co] + sum_{ci,q} f[ci,co,q] * x[b,ci,p+q], geometric product filter
 * first; blade products algebra.py:73-99), the activation against
 * activation.py:142-162, and the error contract (errors.py names in
 * cl_last_error). `--host-only` runs the checks that need no GPU.
 * Test infrastructure: built and run by tests/test_capi_c.py.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "clifford_b200.h"

static int fails = 0;
#define CHECK(c, ...) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
  fprintf(stderr, __VA_ARGS__); fprintf(stderr, "\n"); ++fails; } } while (0)

/* e_I e_J = sign * prod_{i in I&J} g_i * e_{I^J}, sign = (-1)^swaps (algebra.py:73-99) */
static double blade_coeff(int i, int j, const int* g, int k) {
  int swaps = 0;
  for (int s = 1; s < k; ++s) swaps += __builtin_popcount((unsigned)((i >> s) & j));
  double c = (swaps & 1) ? -1.0 : 1.0;
  for (int a = 0; a < k; ++a)
    if ((i & j) >> a & 1) c *= g[a];
  return c;
}

static double lcg(unsigned long long* s) { /* uniform in [-1, 1) */
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((double)(*s >> 11) / 9007199254740992.0) * 2.0 - 1.0;
}

/* fp64 direct conv with zero padding pad (same = (df-1)/2, valid = 0) */
static void conv_ref(const float* x, const float* f, const float* bias, const int* g, int k, int B, int Ci, int Co,
                     int d, int df, int pad, double* y) {
  const int nb = 1 << k, dout = d + 2 * pad - df + 1;
  int P = 1, Q = 1, Po = 1;
  for (int a = 0; a < k; ++a) { P *= d; Q *= df; Po *= dout; }
  for (int b = 0; b < B; ++b)
    for (int co = 0; co < Co; ++co)
      for (int p = 0; p < Po; ++p) {
        int oc[3] = {0, 0, 0}, r = p;
        for (int a = k - 1; a >= 0; --a) { oc[a] = r % dout; r /= dout; }
        for (int t = 0; t < nb; ++t) {
          double acc = bias[t * Co + co];
          for (int ci = 0; ci < Ci; ++ci)
            for (int q = 0; q < Q; ++q) {
              int qc[3] = {0, 0, 0}, rq = q, ip = 0, inside = 1;
              for (int a = k - 1; a >= 0; --a) { qc[a] = rq % df; rq /= df; }
              for (int a = 0; a < k; ++a) {
                const int c = oc[a] + qc[a] - pad;
                if (c < 0 || c >= d) inside = 0;
                ip = ip * d + c;
              }
              if (!inside) continue;
              for (int j = 0; j < nb; ++j) {
                const int i = t ^ j; /* filter blade */
                const double cf = blade_coeff(i, j, g, k);
                if (cf == 0.0) continue;
                acc += cf * f[((i * Ci + ci) * Co + co) * Q + q] * x[((b * Ci + ci) * P + ip) * nb + j];
              }
            }
          y[((b * Co + co) * Po + p) * nb + t] = acc;
        }
      }
}

static void conv_case(const int* g, int k, int B, int Ci, int Co, int d, int df, int padding) {
  const int nb = 1 << k, pad = padding ? (df - 1) / 2 : 0, dout = d + 2 * pad - df + 1;
  int P = 1, Q = 1, Po = 1;
  for (int a = 0; a < k; ++a) { P *= d; Q *= df; Po *= dout; }
  const size_t nx = (size_t)B * Ci * P * nb, nf = (size_t)nb * Ci * Co * Q, ny = (size_t)B * Co * Po * nb;
  float* x = malloc(nx * 4); float* f = malloc(nf * 4); float* bias = malloc((size_t)nb * Co * 4);
  float* y = malloc(ny * 4); double* ref = malloc(ny * 8);
  unsigned long long s = 42;
  for (size_t i = 0; i < nx; ++i) x[i] = (float)lcg(&s);
  for (size_t i = 0; i < nf; ++i) f[i] = (float)(lcg(&s) / sqrt((double)Ci * nb * Q));
  for (int i = 0; i < nb * Co; ++i) bias[i] = (float)(0.01 * lcg(&s));
  int32_t g32[3] = {g[0], k > 1 ? g[1] : 0, k > 2 ? g[2] : 0};
  cl_conv* h = NULL;
  int st = cl_conv_create(g32, k, Ci, Co, d, df, padding, CL_PREC_FP32, f, bias, NULL, &h);
  CHECK(st == CL_OK, "cl_conv_create: %s", cl_last_error());
  if (st == CL_OK) {
    st = cl_conv_forward_host(h, x, y, B, NULL);
    CHECK(st == CL_OK, "cl_conv_forward_host: %s", cl_last_error());
    conv_ref(x, f, bias, g, k, B, Ci, Co, d, df, pad, ref);
    double err = 0.0; /* the reference's max_rel_error, floor 1e-2 (bench.py:74-88) */
    for (size_t i = 0; i < ny; ++i) {
      const double e = fabs(y[i] - ref[i]) / (1e-2 + fmax(fabs(y[i]), fabs(ref[i])));
      if (e > err) err = e;
    }
    CHECK(err <= 1e-4, "conv k=%d padding=%d max_rel_error %.3e", k, padding, err);
    printf("conv k=%d g=(%d,%d,%d) B=%d C=%d->%d d=%d df=%d %s: max_rel_error %.2e\n", k, g[0], g32[1], g32[2], B,
           Ci, Co, d, df, padding ? "same" : "valid", err);
    cl_conv_destroy(h);
  }
  free(x); free(f); free(bias); free(y); free(ref);
}

static void act_case(void) {
  /* Mean aggregation over all 4 blades of g=(1,1): out = x * sigmoid(mean_k x_k) (activation.py:142-162) */
  const int B = 3, C = 5, P = 7, nb = 4;
  int32_t g[2] = {1, 1}, ki[4] = {0, 1, 2, 3};
  float x[3 * 5 * 7 * 4], y[3 * 5 * 7 * 4];
  unsigned long long s = 7;
  for (int i = 0; i < B * C * P * nb; ++i) x[i] = (float)(2.0 * lcg(&s));
  cl_act* a = NULL;
  int st = cl_act_create(g, 2, 2, ki, 4, C, NULL, NULL, NULL, &a);
  CHECK(st == CL_OK, "cl_act_create: %s", cl_last_error());
  if (st != CL_OK) return;
  st = cl_act_forward_host(a, x, y, B, P, NULL);
  CHECK(st == CL_OK, "cl_act_forward_host: %s", cl_last_error());
  double err = 0.0;
  for (int m = 0; m < B * C * P; ++m) {
    float sum = 0.f;
    for (int j = 0; j < nb; ++j) sum += x[m * nb + j];
    const double gate = 1.0 / (1.0 + exp(-(double)(sum / 4.f)));
    for (int j = 0; j < nb; ++j) err = fmax(err, fabs(y[m * nb + j] - x[m * nb + j] * gate));
  }
  CHECK(err <= 1e-5, "activation max_abs_error %.3e", err);
  printf("activation Mean (B,C,P,N_B)=(%d,%d,%d,%d): max_abs_error %.2e\n", B, C, P, nb, err);
  cl_act_destroy(a);
}

static void host_only(void) {
  CHECK(strncmp(cl_version(), "clifford_b200", 13) == 0, "version %s", cl_version());
  int32_t bad[2] = {0, 0}, bad2[2] = {1, 2};
  CHECK(cl_validate_signature(bad, 2) == CL_ERR_INVALID_SIGNATURE, "all-zero signature");
  CHECK(strncmp(cl_last_error(), "InvalidSignature", 16) == 0, "last_error %s", cl_last_error());
  CHECK(cl_validate_signature(bad2, 2) == CL_ERR_INVALID_METRIC_VALUE, "metric value 2");
  int32_t g3[3] = {1, -1, 0};
  int t, c, n = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      if (cl_blade_product(i, j, g3, 3, &t, &c) != CL_OK || t != (i ^ j) || c != (int)blade_coeff(i, j, (int[]){1, -1, 0}, 3))
        ++n;
    }
  CHECK(n == 0, "%d blade products differ", n);
  CHECK(cl_schedule_terms(g3, 3) == 48, "schedule terms of (1,-1,0)");
  printf("host-only checks done\n");
}

int main(int argc, char** argv) {
  host_only();
  if (!(argc > 1 && strcmp(argv[1], "--host-only") == 0)) {
    conv_case((int[]){1, 1}, 2, 2, 3, 4, 9, 3, 0);
    conv_case((int[]){1, 1}, 2, 2, 3, 4, 9, 3, 1);
    conv_case((int[]){1, 1, 1}, 3, 2, 3, 2, 6, 3, 1);
    conv_case((int[]){1, -1, 0}, 3, 1, 2, 3, 5, 3, 0);
    act_case();
  }
  printf(fails ? "capi_demo FAILED (%d)\n" : "capi_demo ok\n", fails);
  return fails ? 1 : 0;
}
