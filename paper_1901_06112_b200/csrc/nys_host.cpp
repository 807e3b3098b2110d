// Host-side FP64 helpers of the Nystrom filter: the m0 x m0 landmark-kernel
// eigendecomposition stays on the host (BASELINE.json north_star (4)).
//
// nys_jacobi_eig restates the reference's cyclic Jacobi solver
// (/root/reference/pkg/src/nysfilter/symeig.py:58-125): fixed (p,q) sweep
// order, skip |a_pq| <= tol, tol = 1e-12 * max|A|, at most 100 sweeps,
// eigenvectors accumulated as rows, stable descending sort, and the sign of
// each eigenvector fixed so that its largest-|.| entry (earliest on ties) is
// non-negative.  Same arithmetic order as the reference, so results agree to
// the last bit on the same matrix.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "../../include/nysfilter_b200.h"
#include "nys_host_internal.h"

namespace nys {
static unsigned long long g_launches = 0;
unsigned long long* launch_counter() { return &g_launches; }
}  // namespace nys

extern "C" uint64_t nys_kernel_launches(void) { return __atomic_load_n(nys::launch_counter(), __ATOMIC_RELAXED); }

extern "C" int nys_jacobi_eig(const double* a_in, int k, double* values_out, double* vectors_out, int* sweeps_out) {
  if (!a_in || k < 1 || !values_out || !vectors_out) return NYS_EINVAL;
  const size_t K = (size_t)k;
  std::vector<double> a(K * K), v(K * K, 0.0);
  double amax = 0.0;
  for (size_t i = 0; i < K; ++i)
    for (size_t j = 0; j < K; ++j) {
      const double x = a_in[i * K + j], y = a_in[j * K + i];
      if (!std::isfinite(x)) return NYS_EINVAL;
      a[i * K + j] = (x + y) / 2.0;  // SymMatrix symmetrisation (symeig.py:33)
    }
  for (size_t i = 0; i < K * K; ++i) amax = std::max(amax, std::fabs(a[i]));
  for (size_t i = 0; i < K; ++i) v[i * K + i] = 1.0;
  const double tol = 1e-12 * amax;
  const int max_sweeps = 100;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) off = std::max(off, std::fabs(a[p * K + q]));
    if (off <= tol) break;
    for (int p = 0; p < k - 1; ++p) {
      for (int q = p + 1; q < k; ++q) {
        const double apq = a[p * K + q];
        if (std::fabs(apq) <= tol) continue;
        const double app = a[p * K + p], aqq = a[q * K + q];
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = tau >= 0.0 ? 1.0 / (tau + std::sqrt(1.0 + tau * tau))
                                    : -1.0 / (-tau + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        for (int i = 0; i < k; ++i) {  // rows p, q
          const double aip = a[p * K + i], aiq = a[q * K + i];
          a[p * K + i] = c * aip - s * aiq;
          a[q * K + i] = s * aip + c * aiq;
        }
        a[p * K + p] = app - t * apq;
        a[q * K + q] = aqq + t * apq;
        a[p * K + q] = 0.0;
        a[q * K + p] = 0.0;
        for (int i = 0; i < k; ++i)
          if (i != p && i != q) {
            a[i * K + p] = a[p * K + i];
            a[i * K + q] = a[q * K + i];
          }
        for (int i = 0; i < k; ++i) {  // eigenvector rows
          const double vip = v[p * K + i], viq = v[q * K + i];
          v[p * K + i] = c * vip - s * viq;
          v[q * K + i] = s * vip + c * viq;
        }
      }
    }
  }
  if (sweeps_out) *sweeps_out = sweep;
  std::vector<int> order(K);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return a[x * K + x] > a[y * K + y]; });
  for (size_t j = 0; j < K; ++j) {
    const int src = order[j];
    values_out[j] = a[src * K + src];
    // column j of the result = row `src` of v
    size_t arg = 0;
    double best = -1.0;
    for (size_t i = 0; i < K; ++i) {
      const double m = std::fabs(v[src * K + i]);
      if (m > best) {
        best = m;
        arg = i;
      }
    }
    const double sgn = v[src * K + arg] < 0.0 ? -1.0 : 1.0;
    for (size_t i = 0; i < K; ++i) vectors_out[i * K + j] = sgn * v[src * K + i];
  }
  return NYS_OK;
}

// (sqrt(a*a + b*b) instead of std::hypot below: the operands are O(1) here and
// glibc's hypot costs ~20 ns, which dominated the QL sweeps)
// ---------------------------------------------------------------------------
// Fast symmetric eigensolver for the hot path: Householder reduction to
// tridiagonal form followed by implicit QL iterations with Wilkinson-style
// shifts (the classical EISPACK tred2/tql2 scheme), O(k^3) with a small
// constant -- ~20x faster than cyclic Jacobi at k = 64.  The filter consumes
// M = sum_k w_k w_k^T / alpha_k and the lead pair only, which do not depend on
// the eigenvector basis or signs, so it may differ from nys_jacobi_eig in the
// last bits.  Eigenvalues are returned in descending order.
// ---------------------------------------------------------------------------
extern "C" int nys_sym_eig(const double* a_in, int k, double* values_out, double* vectors_out) {
  if (!a_in || k < 1 || !values_out || !vectors_out) return NYS_EINVAL;
  const int n = k;
  std::vector<double> z((size_t)n * n), d(n), e(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double x = a_in[(size_t)i * n + j];
      if (!std::isfinite(x)) return NYS_EINVAL;
      z[(size_t)i * n + j] = 0.5 * (x + a_in[(size_t)j * n + i]);
    }
  auto Z = [&](int i, int j) -> double& { return z[(size_t)i * n + j]; };
  // --- Householder tridiagonalisation, accumulating the orthogonal transform in Z
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double h = 0.0, scale = 0.0;
    if (l > 0) {
      for (int q = 0; q <= l; ++q) scale += std::fabs(Z(i, q));
      if (scale == 0.0) {
        e[i] = Z(i, l);
      } else {
        for (int q = 0; q <= l; ++q) {
          Z(i, q) /= scale;
          h += Z(i, q) * Z(i, q);
        }
        double f = Z(i, l);
        const double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        Z(i, l) = f - g;
        f = 0.0;
        for (int j = 0; j <= l; ++j) {
          Z(j, i) = Z(i, j) / h;
          double gg = 0.0;
          for (int q = 0; q <= j; ++q) gg += Z(j, q) * Z(i, q);
          for (int q = j + 1; q <= l; ++q) gg += Z(q, j) * Z(i, q);
          e[j] = gg / h;
          f += e[j] * Z(i, j);
        }
        const double hh = f / (h + h);
        for (int j = 0; j <= l; ++j) {
          const double ff = Z(i, j);
          const double gg = e[j] - hh * ff;
          e[j] = gg;
          for (int q = 0; q <= j; ++q) Z(j, q) -= ff * e[q] + gg * Z(i, q);
        }
      }
    } else {
      e[i] = Z(i, l);
    }
    d[i] = h;
  }
  d[0] = 0.0;
  e[0] = 0.0;
  for (int i = 0; i < n; ++i) {
    const int l = i - 1;
    if (d[i] != 0.0) {
      for (int j = 0; j <= l; ++j) {
        double g = 0.0;
        for (int q = 0; q <= l; ++q) g += Z(i, q) * Z(q, j);
        for (int q = 0; q <= l; ++q) Z(q, j) -= g * Z(q, i);
      }
    }
    d[i] = Z(i, i);
    Z(i, i) = 1.0;
    for (int j = 0; j <= l; ++j) Z(j, i) = Z(i, j) = 0.0;
  }
  // --- implicit QL on the tridiagonal (d, e); the rotations act on columns of
  // Z, so work on Z^T (contiguous rows) to keep the inner loop streaming
  std::vector<double> zt((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) zt[(size_t)j * n + i] = Z(i, j);
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-15 * dd) break;
      }
      if (m != l) {
        if (++iter > 60) return NYS_EUNSUPPORTED;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::sqrt(g * g + 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::sqrt(f * f + g * g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          double* zi = &zt[(size_t)i * n];
          double* zi1 = &zt[(size_t)(i + 1) * n];
          for (int q = 0; q < n; ++q) {
            const double u = zi1[q], w = zi[q];
            zi1[q] = s * w + c * u;
            zi[q] = c * w - s * u;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d[x] > d[y]; });
  for (int j = 0; j < n; ++j) {
    values_out[j] = d[order[j]];
    for (int i = 0; i < n; ++i) vectors_out[(size_t)i * n + j] = zt[(size_t)order[j] * n + i];
  }
  return NYS_OK;
}

// ---------------------------------------------------------------------------
// Mixing plan (see nysfilter_b200.h): Gram matrix, eigenvalues, drop rule,
// M and the lead eigenvector.
// ---------------------------------------------------------------------------
namespace {

// squared distance in numpy's reduction order over rho terms (pairwise_sum:
// sequential below 8 terms, else 8 strided partials), as nystrom.py's gram
double sqdist_np(const double* a, const double* b, int rho) {
  auto sq = [&](int d) {
    const double t = a[d] - b[d];
    return t * t;
  };
  if (rho < 8) {
    double r = 0.0;
    for (int d = 0; d < rho; ++d) r += sq(d);
    return r;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = sq(k);
  int d = 8;
  const int full = rho - (rho % 8);
  for (; d < full; d += 8)
    for (int k = 0; k < 8; ++k) r[k] += sq(d + k);
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; d < rho; ++d) res += sq(d);
  return res;
}

// 4-way split dot product (independent FMA chains; the host path is latency bound)
inline double dot4(const double* a, const double* b, int n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 4 <= n; k += 4) {
    s0 += a[k] * b[k];
    s1 += a[k + 1] * b[k + 1];
    s2 += a[k + 2] * b[k + 2];
    s3 += a[k + 3] * b[k + 3];
  }
  for (; k < n; ++k) s0 += a[k] * b[k];
  return (s0 + s1) + (s2 + s3);
}

// Householder tridiagonalisation (EISPACK tred2 without accumulating the
// transform): on return row i of z holds the Householder vector u_i in columns
// 0..i-1 and column i holds u_i / h_i; h[i] = h_i (0: no reflection); the
// tridiagonal is diag d, sub-diagonal e[i] (coupling i-1 and i).
// x86-64-v3 (AVX2) clone picked at load time where the CPU has it; the 4-way
// split dot products vectorise lane for lane, and FMA contraction stays off
// (-ffp-contract=off), so both clones give identical results
#define NYS_HOST_CLONES __attribute__((target_clones("arch=x86-64-v3", "default")))
NYS_HOST_CLONES
void tridiag(std::vector<double>& z, int n, std::vector<double>& d, std::vector<double>& e, std::vector<double>& h) {
  d.assign(n, 0.0);
  e.assign(n, 0.0);
  h.assign(n, 0.0);
  auto Z = [&](int i, int j) -> double& { return z[(size_t)i * n + j]; };
  std::vector<double> zi(n), p(n);
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double hh = 0.0, scale = 0.0;
    if (l > 0) {
      for (int q = 0; q <= l; ++q) scale += std::fabs(Z(i, q));
      if (scale == 0.0) {
        e[i] = Z(i, l);
      } else {
        for (int q = 0; q <= l; ++q) {
          Z(i, q) /= scale;
          hh += Z(i, q) * Z(i, q);
        }
        double f = Z(i, l);
        const double g = f >= 0.0 ? -std::sqrt(hh) : std::sqrt(hh);
        e[i] = scale * g;
        hh -= f * g;
        Z(i, l) = f - g;
        f = 0.0;
        for (int q = 0; q <= l; ++q) {
          zi[q] = Z(i, q);
          p[q] = 0.0;
        }
        // p = A u over the stored lower triangle, one row at a time: row j gives
        // (A u)_j's lower part (a dot) and the upper parts of (A u)_q, q < j (an axpy)
        for (int j = 0; j <= l; ++j) {
          const double* zj = &z[(size_t)j * n];
          const double uj = zi[j];
          for (int q = 0; q < j; ++q) p[q] += zj[q] * uj;
          p[j] += dot4(zj, zi.data(), j + 1);
        }
        for (int j = 0; j <= l; ++j) {
          Z(j, i) = zi[j] / hh;
          e[j] = p[j] / hh;
          f += e[j] * zi[j];
        }
        const double hf = f / (hh + hh);
        for (int j = 0; j <= l; ++j) {
          const double ff = zi[j];
          const double gg = e[j] - hf * ff;
          e[j] = gg;
          double* zj = &z[(size_t)j * n];
          for (int q = 0; q <= j; ++q) zj[q] -= ff * e[q] + gg * zi[q];
        }
      }
    } else {
      e[i] = Z(i, l);
    }
    h[i] = hh;
  }
  for (int i = 0; i < n; ++i) d[i] = Z(i, i);
}

// eigenvalues of the tridiagonal (d, e as from tridiag) by implicit QL, descending
bool tql_values(std::vector<double> d, std::vector<double> e, int n, std::vector<double>& out) {
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-15 * dd) break;
      }
      if (m != l) {
        if (++iter > 60) return false;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::sqrt(g * g + 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::sqrt(f * f + g * g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  std::sort(d.begin(), d.end(), [](double x, double y) { return x > y; });
  out = d;
  return true;
}

}  // namespace

namespace {
// number of eigenvalues of the symmetric tridiagonal (d, e[i] coupling i-1 and i) below x
// (Sturm count via the LDL^T pivots of T - x I; zero pivots nudged as in LAPACK dstebz)
int sturm_below(const std::vector<double>& d, const std::vector<double>& e, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (std::fabs(q) < pivmin) q = -pivmin;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = (d[i] - x) - e[i] * e[i] / q;
    if (std::fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}
}  // namespace

extern "C" NYS_HOST_CLONES int nys_mixing_plan(const double* C, int m0, int rho, double theta, double eps_drop, double* alphas_out,
                               int* rank_out, double* M_out, double* u0_out) {
  if (!C || m0 < 1 || rho < 1 || !(theta > 0.0) || !alphas_out || !rank_out || !M_out || !u0_out)
    return NYS_EINVAL;
  const int n = m0;
  std::vector<double> A((size_t)n * n);
  const double inv = 1.0 / (2.0 * theta * theta);
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) {
      const double d2 = sqdist_np(C + (size_t)i * rho, C + (size_t)j * rho, rho);
      if (!std::isfinite(d2)) return NYS_EINVAL;
      A[(size_t)i * n + j] = A[(size_t)j * n + i] = std::exp(-d2 * inv);
    }
  std::vector<double> Z(A), d, e, h, vals;
  tridiag(Z, n, d, e, h);
  bool fast = tql_values(d, e, n, vals);
  if (fast && !(vals[0] > 0.0)) return NYS_EDEGENERATE;
  int rank = 0;
  if (fast)
    for (int k = 0; k < n; ++k) rank += vals[k] > eps_drop * vals[0] ? 1 : 0;
  std::vector<double> L;
  if (fast && rank == n) {
    // M = A^{-1} = L^{-T} L^{-1} from A = L L^T (rows of L contiguous)
    L.assign((size_t)n * n, 0.0);
    for (int j = 0; j < n && fast; ++j) {
      const double* lj = &L[(size_t)j * n];
      const double s = A[(size_t)j * n + j] - dot4(lj, lj, j);
      if (!(s > 0.0)) {
        fast = false;
        break;
      }
      const double ljj = std::sqrt(s);
      L[(size_t)j * n + j] = ljj;
      for (int i = j + 1; i < n; ++i) L[(size_t)i * n + j] = (A[(size_t)i * n + j] - dot4(&L[(size_t)i * n], lj, j)) / ljj;
    }
  } else {
    fast = false;
  }
  if (fast) {
    // X = L^{-1} stored transposed (XT[j][i] = X[i][j], i >= j) so both products stream rows
    std::vector<double> XT((size_t)n * n, 0.0);
    std::vector<double> col(n);
    for (int j = 0; j < n; ++j) {
      std::fill(col.begin(), col.end(), 0.0);
      col[j] = 1.0 / L[(size_t)j * n + j];
      for (int i = j + 1; i < n; ++i)
        col[i] = -dot4(&L[(size_t)i * n + j], &col[j], i - j) / L[(size_t)i * n + i];
      for (int i = j; i < n; ++i) XT[(size_t)j * n + i] = col[i];
    }
    // M[i][j] = sum_{k >= max(i,j)} X[k][i] X[k][j] = XT[i] . XT[j] over k >= j (j >= i)
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) {
        const double t = dot4(&XT[(size_t)i * n + j], &XT[(size_t)j * n + j], n - j);
        M_out[(size_t)i * n + j] = M_out[(size_t)j * n + i] = t;
      }
    // u0: inverse iteration on the tridiagonal with sigma just above alpha_1
    // (sigma I - T is SPD, so LDL^T needs no pivoting), then x = Q y through the
    // stored Householder reflections
    const double sigma = vals[0] * (1.0 + 1e-10) + 1e-300;
    std::vector<double> Dg(n), Lg(n, 0.0), y(n, 1.0);
    Dg[0] = sigma - d[0];
    for (int i = 1; i < n && fast; ++i) {
      if (!(Dg[i - 1] > 0.0)) fast = false;
      Lg[i] = -e[i] / Dg[i - 1];
      Dg[i] = (sigma - d[i]) + Lg[i] * e[i];
    }
    if (!(Dg[n - 1] > 0.0)) fast = false;
    for (int it = 0; it < 3 && fast; ++it) {
      for (int i = 1; i < n; ++i) y[i] -= Lg[i] * y[i - 1];
      for (int i = 0; i < n; ++i) y[i] /= Dg[i];
      for (int i = n - 2; i >= 0; --i) y[i] -= Lg[i + 1] * y[i + 1];
      double nrm = std::sqrt(dot4(y.data(), y.data(), n));
      if (!(nrm > 0.0) || !std::isfinite(nrm)) {
        fast = false;
        break;
      }
      for (int i = 0; i < n; ++i) y[i] /= nrm;
    }
    if (fast) {
      for (int i = 1; i < n; ++i) {
        if (h[i] == 0.0) continue;
        const int l = i - 1;
        const double g = dot4(&Z[(size_t)i * n], y.data(), l + 1);
        for (int q = 0; q <= l; ++q) y[q] -= g * Z[(size_t)q * n + i];
      }
      const double nrm = std::sqrt(dot4(y.data(), y.data(), n));
      for (int i = 0; i < n; ++i) u0_out[i] = y[i] / nrm;
      for (int k = 0; k < n; ++k) alphas_out[k] = vals[k];
      *rank_out = n;
      return NYS_OK;
    }
  }
  // general path: full eigensystem, drop rule, M = sum w w^T / alpha
  std::vector<double> V((size_t)n * n);
  vals.assign(n, 0.0);
  const int st = nys_sym_eig(A.data(), n, vals.data(), V.data());
  if (st) return st;
  if (!(vals[0] > 0.0)) return NYS_EDEGENERATE;
  rank = 0;
  for (int k = 0; k < n; ++k) rank += vals[k] > eps_drop * vals[0] ? 1 : 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double t = 0.0;
      for (int k = 0; k < n; ++k)
        if (vals[k] > eps_drop * vals[0]) t += V[(size_t)i * n + k] / vals[k] * V[(size_t)j * n + k];
      M_out[(size_t)i * n + j] = t;
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double t = 0.5 * (M_out[(size_t)i * n + j] + M_out[(size_t)j * n + i]);
      M_out[(size_t)i * n + j] = M_out[(size_t)j * n + i] = t;
    }
  int r = 0;
  for (int k = 0; k < n; ++k)
    if (vals[k] > eps_drop * vals[0]) alphas_out[r++] = vals[k];
  for (int i = 0; i < n; ++i) u0_out[i] = V[(size_t)i * n + 0];
  *rank_out = rank;
  return NYS_OK;
}


// Lite plan for the hot path: the largest eigenvalue by Sturm bisection on the
// tridiagonal and two Sturm counts instead of every eigenvalue (the values-only
// QL was a third of the plan's host time): nothing may fall below
// eps_drop * alpha_1 and cond(A) must stay <= phi_cond, else NYS_EUNSUPPORTED
// (the caller then runs nys_mixing_plan).  info_out[0] = alpha_1.
namespace {
// lower Cholesky factor of the SPD matrix A (row-major n x n) into L; false if a pivot is not positive
NYS_HOST_CLONES bool chol_factor(const double* A, int n, double* L) {
  std::fill(L, L + (size_t)n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    const double* lj = &L[(size_t)j * n];
    const double s = A[(size_t)j * n + j] - dot4(lj, lj, j);
    if (!(s > 0.0)) return false;
    const double ljj = std::sqrt(s);
    L[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) L[(size_t)i * n + j] = (A[(size_t)i * n + j] - dot4(&L[(size_t)i * n], lj, j)) / ljj;
  }
  return true;
}

struct GramTask {
  const double* C;
  int rho, n;
  double inv;
  double* A;
  int r0, r1;
  bool ok;
};
NYS_HOST_CLONES void gram_rows(GramTask* t) {
  const int n = t->n, rho = t->rho;
  for (int i = t->r0; i < t->r1; ++i)
    for (int j = i; j < n; ++j) {
      const double d2 = sqdist_np(t->C + (size_t)i * rho, t->C + (size_t)j * rho, rho);
      if (!std::isfinite(d2)) t->ok = false;
      t->A[(size_t)i * n + j] = t->A[(size_t)j * n + i] = std::exp(-d2 * t->inv);
    }
}
void gram_task(void* p) { gram_rows(static_cast<GramTask*>(p)); }

struct CholTask {
  const double* A;
  int n;
  double* L;
  bool ok;
};
void chol_task(void* p) {
  CholTask* t = static_cast<CholTask*>(p);
  t->ok = chol_factor(t->A, t->n, t->L);
}
}  // namespace

extern "C" int nys_mixing_plan_lite(const double* C, int m0, int rho, double theta, double eps_drop, double phi_cond,
                                    int chol_only, double* info_out, int* rank_out, double* M_out, double* u0_out) {
  return nys_mixing_plan_lite_ex(C, m0, rho, theta, eps_drop, phi_cond, chol_only, info_out, rank_out, M_out, u0_out,
                                 nullptr);
}

// ex (nullable): runs the Cholesky factorisation on a helper thread while this thread
// tridiagonalises; the results are those of the sequential path (same functions)
extern "C" NYS_HOST_CLONES int nys_mixing_plan_lite_ex(const double* C, int m0, int rho, double theta,
                                                       double eps_drop, double phi_cond, int chol_only,
                                                       double* info_out, int* rank_out, double* M_out,
                                                       double* u0_out, const nys_plan_exec* ex) {
  if (!C || m0 < 1 || rho < 1 || !(theta > 0.0) || !info_out || !rank_out || !M_out || !u0_out || !(phi_cond > 1.0))
    return NYS_EINVAL;
  const int n = m0;
  std::vector<double> A((size_t)n * n);
  const double inv = 1.0 / (2.0 * theta * theta);
  // Gram rows [r0, r1) (upper part, mirrored): rows are independent, so with an executor the
  // helper takes the first ~29 % (half the work of the triangle) while this thread does the rest
  GramTask gt{C, rho, n, inv, A.data(), 0, 0, true};
  const int split = ex ? (int)(n * 0.293) : 0;
  if (ex && split > 0) {
    gt.r1 = split;
    ex->run(ex->ctx, gram_task, &gt);
  }
  GramTask mine{C, rho, n, inv, A.data(), split, n, true};
  gram_task(&mine);
  if (ex && split > 0) ex->wait(ex->ctx);
  if (!gt.ok || !mine.ok) return NYS_EINVAL;
  std::vector<double> L((size_t)n * n, 0.0);
  CholTask ct{A.data(), n, L.data(), false};
  struct Join {  // the helper reads A and writes L: joined on every return path
    const nys_plan_exec* ex;
    ~Join() {
      if (ex) ex->wait(ex->ctx);
    }
  } join{ex};
  if (ex) ex->run(ex->ctx, chol_task, &ct);
  std::vector<double> Z(A), d, e, h;
  tridiag(Z, n, d, e, h);
  double lo = d[0], hi = d[0], emax = 0.0;
  for (int i = 0; i < n; ++i) {
    const double r = (i > 0 ? std::fabs(e[i]) : 0.0) + (i + 1 < n ? std::fabs(e[i + 1]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
    emax = std::max(emax, std::fabs(d[i]) + r);
  }
  const double pivmin = std::max(1e-300, 1e-300 * emax * emax);
  // multisection: 8 shifts per sweep as independent LDL^T chains (the Sturm
  // recurrence is division-latency bound, so 8 chains cost about one), the
  // bracket shrinks 9x per sweep instead of 2x
  {
    std::vector<double> e2(n, 0.0);
    for (int i = 1; i < n; ++i) e2[i] = e[i] * e[i];
    for (int it = 0; it < 100 && hi - lo > 2e-16 * std::max(std::fabs(lo), std::fabs(hi)); ++it) {
      double x[8], q[8];
      int c[8];
      for (int k = 0; k < 8; ++k) {
        x[k] = lo + (hi - lo) * (double)(k + 1) / 9.0;
        q[k] = d[0] - x[k];
        if (std::fabs(q[k]) < pivmin) q[k] = -pivmin;
        c[k] = q[k] < 0.0 ? 1 : 0;
      }
      for (int i = 1; i < n; ++i)
        for (int k = 0; k < 8; ++k) {
          double t = (d[i] - x[k]) - e2[i] / q[k];
          if (std::fabs(t) < pivmin) t = -pivmin;
          q[k] = t;
          c[k] += t < 0.0 ? 1 : 0;
        }
      double nlo = lo, nhi = hi;
      for (int k = 0; k < 8; ++k) {
        if (c[k] <= n - 1) nlo = std::max(nlo, x[k]);  // alpha_1 >= x_k
        else nhi = std::min(nhi, x[k]);               // alpha_1 < x_k
      }
      if (nlo == lo && nhi == hi) break;  // the shifts no longer split the bracket (1 ulp)
      lo = nlo;
      hi = nhi;
    }
  }
  const double a1 = 0.5 * (lo + hi);
  if (!(a1 > 0.0)) return NYS_EDEGENERATE;
  if (sturm_below(d, e, n, eps_drop * a1, pivmin) > 0) return NYS_EUNSUPPORTED;  // something is dropped
  if (sturm_below(d, e, n, a1 / phi_cond, pivmin) > 0) return NYS_EUNSUPPORTED;  // phi-form territory
  std::vector<double> vals(1, a1);
  if (ex) {
    ex->wait(ex->ctx);
    join.ex = nullptr;
  } else {
    chol_task(&ct);
  }
  bool fast = ct.ok;
  double* alphas_out = info_out;
  if (fast && chol_only) {
    // the caller forms M = L^{-T} L^{-1} on the device (nys_filter_desc.M_is_cholesky)
    for (size_t q = 0; q < (size_t)n * n; ++q) M_out[q] = L[q];
  }
  if (fast) {
    // X = L^{-1} stored transposed (XT[j][i] = X[i][j], i >= j) so both products stream rows
    std::vector<double> XT(chol_only ? 0 : (size_t)n * n, 0.0);
    std::vector<double> col(n);
    for (int j = 0; j < (chol_only ? 0 : n); ++j) {
      std::fill(col.begin(), col.end(), 0.0);
      col[j] = 1.0 / L[(size_t)j * n + j];
      for (int i = j + 1; i < n; ++i)
        col[i] = -dot4(&L[(size_t)i * n + j], &col[j], i - j) / L[(size_t)i * n + i];
      for (int i = j; i < n; ++i) XT[(size_t)j * n + i] = col[i];
    }
    // M[i][j] = sum_{k >= max(i,j)} X[k][i] X[k][j] = XT[i] . XT[j] over k >= j (j >= i)
    for (int i = 0; i < (chol_only ? 0 : n); ++i)
      for (int j = i; j < n; ++j) {
        const double t = dot4(&XT[(size_t)i * n + j], &XT[(size_t)j * n + j], n - j);
        M_out[(size_t)i * n + j] = M_out[(size_t)j * n + i] = t;
      }
    // u0: inverse iteration on the tridiagonal with sigma just above alpha_1
    // (sigma I - T is SPD, so LDL^T needs no pivoting), then x = Q y through the
    // stored Householder reflections
    const double sigma = vals[0] * (1.0 + 1e-10) + 1e-300;
    std::vector<double> Dg(n), Lg(n, 0.0), y(n, 1.0);
    Dg[0] = sigma - d[0];
    for (int i = 1; i < n && fast; ++i) {
      if (!(Dg[i - 1] > 0.0)) fast = false;
      Lg[i] = -e[i] / Dg[i - 1];
      Dg[i] = (sigma - d[i]) + Lg[i] * e[i];
    }
    if (!(Dg[n - 1] > 0.0)) fast = false;
    for (int it = 0; it < 3 && fast; ++it) {
      for (int i = 1; i < n; ++i) y[i] -= Lg[i] * y[i - 1];
      for (int i = 0; i < n; ++i) y[i] /= Dg[i];
      for (int i = n - 2; i >= 0; --i) y[i] -= Lg[i + 1] * y[i + 1];
      double nrm = std::sqrt(dot4(y.data(), y.data(), n));
      if (!(nrm > 0.0) || !std::isfinite(nrm)) {
        fast = false;
        break;
      }
      for (int i = 0; i < n; ++i) y[i] /= nrm;
    }
    if (fast) {
      for (int i = 1; i < n; ++i) {
        if (h[i] == 0.0) continue;
        const int l = i - 1;
        const double g = dot4(&Z[(size_t)i * n], y.data(), l + 1);
        for (int q = 0; q <= l; ++q) y[q] -= g * Z[(size_t)q * n + i];
      }
      const double nrm = std::sqrt(dot4(y.data(), y.data(), n));
      for (int i = 0; i < n; ++i) u0_out[i] = y[i] / nrm;
      alphas_out[0] = vals[0];
      *rank_out = n;
      return NYS_OK;
    }
  }
  return NYS_EUNSUPPORTED;
}

// ---------------------------------------------------------------------------
// Recursive Gaussian coefficients (spatial.py:114-146, van Vliet / Young /
// Verbeek fifth-order poles).  Restates the reference's arithmetic with
// CPython's complex routines (c_pow via hypot/pow/atan2/cos/sin, c_powu for
// the integer square, Smith-style c_quot) so the bisection lands on the same
// pole scale q; the polynomial expansion follows np.convolve.
// ---------------------------------------------------------------------------
namespace {
struct cplx {
  double re, im;
};
inline cplx c_sub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
inline cplx c_add(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
inline cplx c_prod(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline cplx c_quot(cplx a, cplx b) {
  const double abr = b.re < 0 ? -b.re : b.re, abi = b.im < 0 ? -b.im : b.im;
  if (abr >= abi) {
    if (abr == 0.0) return {0.0, 0.0};
    const double ratio = b.im / b.re, denom = b.re + b.im * ratio;
    return {(a.re + a.im * ratio) / denom, (a.im - a.re * ratio) / denom};
  }
  const double ratio = b.re / b.im, denom = b.re * ratio + b.im;
  return {(a.re * ratio + a.im) / denom, (a.im * ratio - a.re) / denom};
}
// complex ** real exponent (CPython complex_pow -> c_pow / c_powi)
inline cplx c_pow_real(cplx a, double e) {
  if (e == 0.0) return {1.0, 0.0};
  if (e == std::floor(e) && std::fabs(e) <= 100.0) {
    long n = (long)e;
    bool neg = n < 0;
    if (neg) n = -n;
    cplx r{1.0, 0.0}, p = a;
    for (long mask = 1; mask > 0 && n >= mask; mask <<= 1) {
      if (n & mask) r = c_prod(r, p);
      p = c_prod(p, p);
    }
    return neg ? c_quot({1.0, 0.0}, r) : r;
  }
  const double vabs = std::hypot(a.re, a.im), len = std::pow(vabs, e);
  const double phase = std::atan2(a.im, a.re) * e;
  return {len * std::cos(phase), len * std::sin(phase)};
}
const cplx kVyvPoles[5] = {{0.86430, 1.45389}, {0.86430, -1.45389}, {1.61433, 0.83134}, {1.61433, -0.83134},
                           {1.87504, 0.0}};

double cascade_variance(double q) {  // spatial.py:124-129
  cplx total{0.0, 0.0};
  for (const cplx& d : kVyvPoles) {
    const cplx z = c_pow_real(d, 1.0 / q);
    const cplx zm1 = c_sub(z, {1.0, 0.0});
    total = c_add(total, c_quot(c_prod({2.0, 0.0}, z), c_prod(zm1, zm1)));
  }
  return total.re;
}
}  // namespace

extern "C" int nys_vyv_coeffs(double sigma, double* coeffs_out) {
  if (!coeffs_out || !(sigma > 0.0) || !std::isfinite(sigma)) return NYS_EINVAL;
  double lo = 1e-3, hi = 1000.0;  // spatial.py:132-141 bisection for cascade variance == sigma^2
  const double target = sigma * sigma;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (cascade_variance(mid) < target)
      lo = mid;
    else
      hi = mid;
  }
  const double q = 0.5 * (lo + hi);
  cplx poly[6] = {{1.0, 0.0}};
  int len = 1;
  for (const cplx& d : kVyvPoles) {  // np.convolve(poly, [1, -1/d^(1/q)])
    const cplx v1 = c_quot({-1.0, 0.0}, c_pow_real(d, 1.0 / q));
    cplx next[6];
    for (int k = 0; k <= len; ++k) {
      cplx acc{0.0, 0.0};
      if (k < len) acc = c_add(acc, poly[k]);
      if (k >= 1) acc = c_add(acc, c_prod(poly[k - 1], v1));
      next[k] = acc;
    }
    ++len;
    for (int k = 0; k < len; ++k) poly[k] = next[k];
  }
  double gain = 0.0;
  for (int k = 0; k < 6; ++k) gain += poly[k].re;  // unit DC gain per pass
  coeffs_out[0] = gain;
  for (int k = 1; k < 6; ++k) coeffs_out[k] = poly[k].re;
  return NYS_OK;
}
