// Library-internal host entry points (not part of the public C ABI in include/).
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

// Runs fn(arg) on a helper thread (run) and joins it (wait); used by the in-stream
// plan's worker to factor A while it tridiagonalises.
typedef struct nys_plan_exec {
  void (*run)(void* ctx, void (*fn)(void*), void* arg);
  void (*wait)(void* ctx);
  void* ctx;
} nys_plan_exec;

// nys_mixing_plan_lite with an optional executor (NULL: sequential, identical results)
int nys_mixing_plan_lite_ex(const double* C, int m0, int rho, double theta, double eps_drop, double phi_cond,
                            int chol_only, double* info_out, int* rank_out, double* M_out, double* u0_out,
                            const nys_plan_exec* ex);

#ifdef __cplusplus
}
#endif
