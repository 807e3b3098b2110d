"""ctypes binding of the C ABI in ``include/nysfilter_b200.h``.

The library is built in-tree by ``paper_1901_06112_b200.build`` and loaded
from ``paper_1901_06112_b200/_lib``.  There is deliberately no fallback: if the
library is missing or the GPU is absent, calls fail loudly.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libnysfilter_b200.so"

NYS_OK = 0
NYS_EINVAL = 1
NYS_EUNSUPPORTED = 2
NYS_EDEGENERATE = 3
NYS_ECUDA = 1000
NYS_SPATIAL_BOX = 0
NYS_SPATIAL_GAUSSIAN_FIR = 1
NYS_SPATIAL_GAUSSIAN_RECURSIVE = 2
NYS_MAX_RADIUS = 64
NYS_MAX_M0 = 256
NYS_MAX_RHO = 64        # register-resident guides (the fast kernels)
NYS_MAX_RHO_WIDE = 1024  # generic paths beyond (step-wise k-means, features as planes before K2)
NYS_MAX_CHANNELS = 64
NYS_MAX_CHANNELS_WIDE = 511


class NativeError(RuntimeError):
    """A C-ABI entry point returned a non-zero status."""


class FilterDesc(C.Structure):
    """Mirror of ``nys_filter_desc``."""

    _fields_ = [
        ("n", C.c_int), ("rho", C.c_int), ("H", C.c_int), ("W", C.c_int),
        ("guide_kind", C.c_int), ("spatial_kind", C.c_int), ("radius", C.c_int),
        ("sigma", C.c_double), ("m0", C.c_int), ("theta", C.c_double),
        ("centroids", C.POINTER(C.c_double)), ("M", C.POINTER(C.c_double)),
        ("u0", C.POINTER(C.c_double)), ("alpha0", C.c_double), ("eps_den", C.c_double),
        ("row_lo", C.c_int), ("row_hi", C.c_int), ("phi_form", C.c_int), ("M_is_cholesky", C.c_int),
        ("out_f64", C.c_int),
    ]


class PlanResult(C.Structure):
    """Mirror of ``nys_plan_result``."""

    _fields_ = [("status", C.c_int), ("rank", C.c_int), ("alpha0", C.c_double), ("eps_den", C.c_double),
                ("host_us", C.c_double)]


_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_S = C.c_size_t
_D = C.c_double

_SIGS = {
    "nys_abi_version": (_I, []),
    "nys_kernel_launches": (C.c_uint64, []),
    "nys_kmeans_workspace_bytes": (_S, [_L, _I, _I]),
    "nys_kmeans_run": (_I, [_P, _L, _L, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P, _P, _P, _S, _P]),
    "nys_kmeans_run_seeded": (_I, [_P, _L, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _S, _P]),
    "nys_kmeanspp_update": (_I, [_P, _L, _L, _I, _P, _I, _P, _P, _P, _S, _P]),
    "nys_kmeanspp_pick": (_I, [_P, _L, _D, _P, _P, _S, _P]),
    "nys_kmeans_assign": (_I, [_P, _L, _L, _I, _P, _I, _P, _I, _P, _P, _S, _P]),
    "nys_kmeans_exact": (_I, [_P, _L, _L, _I, _P, _I, _P, _P, _P, _S, _P]),
    "nys_kmeans_farthest": (_I, [_P, _L, _L, _I, _P, _I, _P, _P, _I, _P, _P, _S, _P]),
    "nys_gather_point": (_I, [_P, _L, _I, _L, _P, _P]),
    "nys_kmeans_state_init": (_I, [_P, _S, _L, _I, _I, _P]),
    "nys_kmeans_state_read": (_I, [_P, _L, _I, _I, _P, _P]),
    "nys_kmeanspp_owner_pick": (_I, [_P, _L, _L, _I, _I, _P, _P, _I, _I, _L, _D, _I, _P, _P, _S, _P]),
    "nys_kmeans_lloyd_local": (_I, [_P, _L, _L, _I, _P, _I, _I, _I, _P, _P, _P, _S, _P]),
    "nys_kmeans_lloyd_update": (_I, [_L, _I, _I, _I, _I, _P, _P, _P, _P, _P, _S, _P]),
    "nys_filter_planes_bytes": (_S, [C.POINTER(FilterDesc), _I]),
    "nys_filter_workspace_bytes": (_S, [C.POINTER(FilterDesc)]),
    "nys_filter_workspace_layout": (_I, [C.POINTER(FilterDesc), _P]),
    "nys_filter_plane_row_stride": (_L, [C.POINTER(FilterDesc)]),
    "nys_filter_prepare": (_I, [C.POINTER(FilterDesc), _P, _S, _P]),
    "nys_filter_plan_staging_bytes": (_S, [C.POINTER(FilterDesc)]),
    "nys_filter_plan_async": (_I, [C.POINTER(FilterDesc), _P, _D, _D, _P, _S, _P, _S, _P]),
    "nys_filter_prepare_join": (_I, [C.POINTER(FilterDesc), _P, _P, _P]),
    "nys_filter_plan_result": (_I, [_P, C.POINTER(PlanResult)]),
    "nys_filter_hpass": (_I, [C.POINTER(FilterDesc), _P, _L, _P, _L, _I, _I, _P, _L, _P, _P]),
    "nys_filter_vpass": (_I, [C.POINTER(FilterDesc), _P, _L, _P, _L, _P, _L, _I, _I, _P, _L, _P, _P]),
    "nys_filter_finish": (_I, [C.POINTER(FilterDesc), _P, _L, _P, _L, _P, _L, _P, _P, _P]),
    "nys_filter_stats": (_I, [C.POINTER(FilterDesc), _P, _P, _P]),
    "nys_patch_guide": (_I, [_P, _L, _I, _I, _I, _I, _P, _L, _P]),
    "nys_jacobi_eig": (_I, [_P, _I, _P, _P, C.POINTER(C.c_int)]),
    "nys_sym_eig": (_I, [_P, _I, _P, _P]),
    "nys_device_view": (_I, [_P, C.POINTER(C.c_void_p)]),
    "nys_vyv_coeffs": (_I, [_D, _P]),
    "nys_filter_recursive_scratch_bytes": (_S, [C.POINTER(FilterDesc), _I]),
    "nys_filter_recursive": (_I, [C.POINTER(FilterDesc), _P, _L, _P, _L, _P, _L, _P, _S, _P, _P]),
    "nys_brute_force_filter": (_I, [C.POINTER(FilterDesc), _P, _L, _P, _L, _P, _L, _P]),
    "nys_quality_workspace_bytes": (_S, [_I]),
    "nys_quality_planes": (_I, [_P, _L, _P, _L, _I, _I, _I, _I, _D, _P, _P, _P, _S, _P]),
    "nys_patch_moments_workspace_bytes": (_S, [_I, _I, _I, _I]),
    "nys_patch_moments": (_I, [_P, _L, _I, _I, _I, _I, _P, _P, _P, _S, _P]),
    "nys_pca_project": (_I, [_P, _L, _I, _I, _I, _I, _P, _P, _I, _P, _L, _P]),
    "nys_spatial_planes": (_I, [_P, _P, _L, _I, _I, _I, _D, _I, _P, _P]),
    "nys_mixing_plan_lite": (_I, [_P, _I, _I, _D, _D, _D, _I, _P, C.POINTER(C.c_int), _P, _P]),
    "nys_mixing_plan": (_I, [_P, _I, _I, _D, _D, _P, C.POINTER(C.c_int), _P, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the native library; raises if it is absent."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: run paper_1901_06112_b200.build.build() "
                "(there is no CPU fallback)")
        h = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(rc: int, what: str) -> None:
    if rc == NYS_OK:
        return
    if rc == NYS_EINVAL:
        raise ValueError(f"{what}: invalid argument")
    if rc == NYS_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: configuration not supported by the B200 kernels")
    if rc >= NYS_ECUDA:
        raise NativeError(f"{what}: CUDA error {rc - NYS_ECUDA}")
    raise NativeError(f"{what}: status {rc}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
