// basis.cu -- SURVEY 8f row f4: flop-reducing change of basis.
//
// For non-degenerate signatures whose real Clifford algebra is a full 2x2
// matrix algebra -- Cl(2,0) ~ Cl(1,1) ~ M2(R), Cl(3,0) ~ Cl(1,2) ~ M2(C) --
// a multivector x maps to a 2x2 matrix X = sum_I x_I M_I (M_I = product of
// generator matrices), and the geometric product f x maps to the matrix
// product F X. Left multiplication acts on the two COLUMNS of X
// independently with the same operator R(f), so in the coordinates
//   x' = T x   (T: rows = (column c, component r) of X, entries in {0, +-1},
//               T T^T = 2 I, so x = T^T x' / 2)
// the Clifford conv splits into ncol = 2 independent real GEMMs sharing one
// filter R(f) of size w x w (w = 2 real, 4 for complex entries): half the
// multiply-adds of the expanded N_B x N_B kernel (conv.py:188-202).
//
// find_basis() searches Pauli-type generator assignments for the signature
// and validates the result exactly: T T^T = 2 I and, for every blade e_J,
// T L(e_J) T^T / 2 block-diagonal with identical w x w blocks.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace cl {
namespace {

struct C2 {  // complex 2x2
  double re[2][2], im[2][2];
};

C2 mul(const C2& a, const C2& b) {
  C2 c{};
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k) {
        c.re[i][j] += a.re[i][k] * b.re[k][j] - a.im[i][k] * b.im[k][j];
        c.im[i][j] += a.re[i][k] * b.im[k][j] + a.im[i][k] * b.re[k][j];
      }
  return c;
}

C2 ident() {
  C2 c{};
  c.re[0][0] = c.re[1][1] = 1;
  return c;
}

bool is_scalar(const C2& m, double s) {  // m == s * I
  return m.re[0][0] == s && m.re[1][1] == s && m.re[0][1] == 0 && m.re[1][0] == 0 && m.im[0][0] == 0 &&
         m.im[1][1] == 0 && m.im[0][1] == 0 && m.im[1][0] == 0;
}

bool anticommute(const C2& a, const C2& b) {
  const C2 x = mul(a, b), y = mul(b, a);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      if (x.re[i][j] != -y.re[i][j] || x.im[i][j] != -y.im[i][j]) return false;
  return true;
}

std::vector<C2> candidates(bool real_only, int square) {
  // Pauli matrices s1, s2, s3 (square +I) and i*s1, i*s2, i*s3 (square -I)
  C2 s1{}, s2{}, s3{};
  s1.re[0][1] = s1.re[1][0] = 1;
  s2.im[0][1] = -1;
  s2.im[1][0] = 1;
  s3.re[0][0] = 1;
  s3.re[1][1] = -1;
  auto times_i = [](const C2& a) {
    C2 c{};
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) {
        c.re[i][j] = -a.im[i][j];
        c.im[i][j] = a.re[i][j];
      }
    return c;
  };
  std::vector<C2> all = square > 0 ? std::vector<C2>{s1, s2, s3}
                                   : std::vector<C2>{times_i(s1), times_i(s2), times_i(s3)};
  std::vector<C2> out;
  for (auto& m : all) {
    bool real = true;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) real = real && m.im[i][j] == 0;
    if (!real_only || real) out.push_back(m);
  }
  return out;
}

// Exact validation of a candidate T (rows = (column, component), ncol = 2
// identical w x w blocks) and fill of the Basis record: T T^T = 2 I, every
// blade's left multiplication block-diagonal with identical blocks, and the
// two-term forms of T and T^T used by the device kernels.
bool validate_and_fill(const int* g, int k, const int (&T)[8][8], int w, Basis* bs) {
  const int nb = 1 << k;
  // T T^T == 2 I
  for (int a = 0; a < nb; ++a)
    for (int b = 0; b < nb; ++b) {
      int d = 0;
      for (int I = 0; I < nb; ++I) d += T[a][I] * T[b][I];
      if (d != (a == b ? 2 : 0)) return false;
    }
  // left multiplication by every blade is block-diagonal with identical blocks
  for (int J = 0; J < nb; ++J) {
    double L[8][8] = {};
    for (int j = 0; j < nb; ++j) L[J ^ j][j] = blade_coeff(J, j, g, k);
    double A[8][8] = {};
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b < nb; ++b) {
        double s = 0;
        for (int x = 0; x < nb; ++x)
          for (int y = 0; y < nb; ++y) s += T[a][x] * L[x][y] * T[b][y];
        A[a][b] = s / 2;
      }
    for (int a = 0; a < nb; ++a)
      for (int b = 0; b < nb; ++b) {
        const int ca = a / w, cb = b / w;
        if (ca != cb && A[a][b] != 0) return false;
        if (ca == cb && A[a][b] != A[a % w][b % w]) return false;
      }
  }
  bs->on = 1;
  bs->ncol = 2;
  bs->w = w;
  for (int a = 0; a < 8; ++a)
    for (int I = 0; I < 8; ++I) bs->T[a * 8 + I] = (int8_t)((a < nb && I < nb) ? T[a][I] : 0);
  // two-term forms of T (rows) and T^T (columns)
  for (int a = 0; a < nb; ++a) {
    int n = 0, m = 0;
    for (int I = 0; I < nb; ++I) {
      if (T[a][I]) {
        if (n == 2) return false;
        bs->fwd[a][n] = (int8_t)I;
        bs->fwd_sgn[a][n++] = (int8_t)T[a][I];
      }
      if (T[I][a]) {
        if (m == 2) return false;
        bs->inv[a][m] = (int8_t)I;
        bs->inv_sgn[a][m++] = (int8_t)T[I][a];
      }
    }
    if (n != 2 || m != 2) return false;
  }
  return true;
}


bool build_and_check(const int* g, int k, const std::vector<C2>& gen, Basis* bs) {
  const int nb = 1 << k;
  const bool cplx = (k == 3);
  const int w = cplx ? 4 : 2;
  std::vector<C2> M(nb);
  for (int I = 0; I < nb; ++I) {
    C2 m = ident();
    for (int bit = 0; bit < k; ++bit)
      if ((I >> bit) & 1) m = mul(m, gen[bit]);
    M[I] = m;
  }
  int T[8][8] = {};
  for (int c = 0; c < 2; ++c)
    for (int r = 0; r < 2; ++r)
      for (int part = 0; part < (cplx ? 2 : 1); ++part) {
        const int s = c * w + r * (cplx ? 2 : 1) + part;
        for (int I = 0; I < nb; ++I) {
          const double v = part ? M[I].im[r][c] : M[I].re[r][c];
          if (v != 0 && v != 1 && v != -1) return false;
          T[s][I] = (int)v;
        }
      }
  return validate_and_fill(g, k, T, w, bs);
}

}  // namespace

// Degenerate k = 3 signature with exactly one null generator e_z whose other
// two generators span M2(R) (Cl(2,0), Cl(1,1)): x = a + b e_z with a, b in
// that M2(R), and since e_z e_z = 0 and e_z c = c^ e_z (grade involution),
//   f x = f_a x_a + (f_a x_b + f_b x_a^) e_z.
// With c^ = E c E^-1 (E = the pair's pseudoscalar matrix) and Z = X_b E, each
// column of (X_a, Z) transforms by the same lower block-triangular operator
// [[F_a, 0], [F_b E, F_a]]: two identical 4 x 4 blocks, half the multiply-adds
// of the 8 x 8 expanded kernel (SURVEY 8f f4 extended to H4's signatures).
// T is assembled from the pair's 2-D basis; the column swap and signs that
// realise Z are searched and the result validated exactly.
static bool find_degenerate_basis(const int* g, int k, Basis* bs) {
  if (k != 3) return false;
  int z = -1, nz = 0;
  for (int i = 0; i < 3; ++i)
    if (g[i] == 0) { z = i; ++nz; }
  if (nz != 1) return false;
  int gi[2], pos[2], n = 0;
  for (int i = 0; i < 3; ++i)
    if (i != z) { pos[n] = i; gi[n++] = g[i]; }
  Basis pb;
  if (!find_basis(gi, 2, &pb)) return false;  // pair must be M2(R)
  auto full = [&](int m) {  // pair blade (2-bit) -> full blade mask
    return ((m & 1) ? (1 << pos[0]) : 0) | ((m & 2) ? (1 << pos[1]) : 0);
  };
  for (int swap = 0; swap < 2; ++swap)
    for (int sg = 0; sg < 16; ++sg) {
      int T[8][8] = {};
      for (int c = 0; c < 2; ++c)
        for (int r = 0; r < 2; ++r) {
          const int sA = c * 4 + r, sB = c * 4 + 2 + r;
          const int sgn = ((sg >> (c * 2 + r)) & 1) ? -1 : 1;
          for (int m = 0; m < 4; ++m) {
            const int I = full(m);
            T[sA][I] = pb.T[(c * 2 + r) * 8 + m];
            // coefficient of e_I e_z = reorder sign * x_{I | z}
            T[sB][I | (1 << z)] = sgn * pb.T[((c ^ swap) * 2 + r) * 8 + m] * blade_coeff(I, 1 << z, g, k);
          }
        }
      if (validate_and_fill(g, k, T, 4, bs)) return true;
    }
  *bs = Basis{};
  return false;
}

bool find_basis(const int* g, int k, Basis* bs) {
  *bs = Basis{};
  if (k != 2 && k != 3) return false;
  for (int i = 0; i < k; ++i)
    if (g[i] == 0) return find_degenerate_basis(g, k, bs);  // not semisimple: see above
  std::vector<std::vector<C2>> cand(k);
  for (int i = 0; i < k; ++i) cand[i] = candidates(k == 2, g[i]);
  std::vector<C2> gen(k);
  // exhaustive over the (at most 3^3) assignments
  int idx[3] = {0, 0, 0};
  while (true) {
    bool ok = true;
    for (int i = 0; i < k && ok; ++i) {
      if (idx[i] >= (int)cand[i].size()) { ok = false; break; }
      gen[i] = cand[i][idx[i]];
      if (!is_scalar(mul(gen[i], gen[i]), (double)g[i])) ok = false;
      for (int j = 0; j < i && ok; ++j) ok = anticommute(gen[i], gen[j]);
    }
    if (ok && build_and_check(g, k, gen, bs)) return true;
    int p = 0;
    while (p < k && ++idx[p] >= (int)cand[p].size()) idx[p++] = 0;
    if (p == k) break;
  }
  *bs = Basis{};
  return false;
}

}  // namespace cl
