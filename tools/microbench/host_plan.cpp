// Stage timing of nys_mixing_plan_lite on this host (Gram, tridiagonalisation,
// bisection for alpha_1, Sturm counts, Cholesky, u0):
//   g++ -O3 -std=c++17 -ffp-contract=off -I include tools/microbench/host_plan.cpp -o /tmp/host_plan
//   /tmp/host_plan centroids.bin m0 rho theta
#include "../../paper_1901_06112_b200/csrc/nys_host.cpp"
#include <chrono>
#include <cstdio>
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  const int n = atoi(argv[2]), rho = atoi(argv[3]);
  const double theta = atof(argv[4]);
  std::vector<double> C((size_t)n * rho);
  FILE* f = fopen(argv[1], "rb");
  if (fread(C.data(), 8, C.size(), f) != C.size()) return 1;
  fclose(f);
  const int R = 2000;
  double tg = 0, tt = 0, tb = 0, tc = 0, tall = 0;
  std::vector<double> A((size_t)n * n), Z, d, e, h, L((size_t)n * n);
  int iters = 0;
  for (int r = 0; r < R; ++r) {
    double t0 = now();
    const double inv = 1.0 / (2.0 * theta * theta);
    for (int i = 0; i < n; ++i)
      for (int j = i; j < n; ++j) A[(size_t)i * n + j] = A[(size_t)j * n + i] = std::exp(-sqdist_np(&C[(size_t)i * rho], &C[(size_t)j * rho], rho) * inv);
    double t1 = now();
    Z = A;
    tridiag(Z, n, d, e, h);
    double t2 = now();
    double lo = d[0], hi = d[0], emax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double rr = (i > 0 ? std::fabs(e[i]) : 0.0) + (i + 1 < n ? std::fabs(e[i + 1]) : 0.0);
      lo = std::min(lo, d[i] - rr); hi = std::max(hi, d[i] + rr); emax = std::max(emax, std::fabs(d[i]) + rr);
    }
    const double pivmin = std::max(1e-300, 1e-300 * emax * emax);
    iters = 0;
    for (int it = 0; it < 200 && hi - lo > 2e-16 * std::max(std::fabs(lo), std::fabs(hi)); ++it, ++iters) {
      const double mid = 0.5 * (lo + hi);
      if (sturm_below(d, e, n, mid, pivmin) <= n - 1) lo = mid; else hi = mid;
    }
    double t3 = now();
    std::fill(L.begin(), L.end(), 0.0);
    for (int j = 0; j < n; ++j) {
      const double* lj = &L[(size_t)j * n];
      const double s = A[(size_t)j * n + j] - dot4(lj, lj, j);
      const double ljj = std::sqrt(s);
      L[(size_t)j * n + j] = ljj;
      for (int i = j + 1; i < n; ++i) L[(size_t)i * n + j] = (A[(size_t)i * n + j] - dot4(&L[(size_t)i * n], lj, j)) / ljj;
    }
    double t4 = now();
    std::vector<double> info(n), M((size_t)n * n), u0(n);
    int rank;
    nys_mixing_plan_lite(C.data(), n, rho, theta, 1e-8, 3e4, 1, info.data(), &rank, M.data(), u0.data());
    double t5 = now();
    if (r >= 100) { tg += t1 - t0; tt += t2 - t1; tb += t3 - t2; tc += t4 - t3; tall += t5 - t4; }
  }
  const double k = R - 100;
  printf("gram %.1f  tridiag %.1f  bisect %.1f (%d it)  chol %.1f  | lite(chol_only) %.1f us\n", tg / k, tt / k, tb / k, iters, tc / k, tall / k);
}
