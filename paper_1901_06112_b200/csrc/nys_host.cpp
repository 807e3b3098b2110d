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
