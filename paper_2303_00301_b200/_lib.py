"""ctypes view of include/auxmc_gpu.h and the loader of libauxmc_b200.so.

The product path has no CPU fallback: if the shared library is missing, or no
sm_100 device is usable, compute entry points raise.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

PKG = pathlib.Path(__file__).resolve().parent
# AUXMC_LIB_PATH: an alternative in-tree build (tools/exp_build.sh kernel experiments)
LIB_PATH = pathlib.Path(os.environ["AUXMC_LIB_PATH"]) if os.environ.get("AUXMC_LIB_PATH") \
    else PKG / "libauxmc_b200.so"

OK, E_DIM, E_FACTOR, E_DEGENERATE, E_CONTRACT, E_CONFIG, E_CUDA, E_ARG, E_WORKSPACE = range(9)
NOISE_STREAM, NOISE_PREDRAWN = 0, 1
SAMPLER_SEQ, SAMPLER_PREFIX, SAMPLER_DNC = 0, 1, 2
KIND = {"lgssm-synthetic": 0, "stochvol": 1, "diffusion-smoothing": 2, "spatio-temporal": 3,
        "grid-1d-test": 4, "lorenz96": 5, "gauss-generic": 6, "test-abort": 7, "test-support": 8,
        "test-collapse": 9}

PD = C.POINTER(C.c_double)
PU8 = C.POINTER(C.c_uint8)
PU64 = C.POINTER(C.c_uint64)
PI = C.POINTER(C.c_int)
PLL = C.POINTER(C.c_longlong)


class Lgssm(C.Structure):
    _fields_ = [("T", C.c_int), ("dx", C.c_int), ("dy", C.c_int), ("m0", C.c_void_p),
                ("P0", C.c_void_p), ("F", C.c_void_p), ("nF", C.c_int), ("b", C.c_void_p),
                ("nb", C.c_int), ("Q", C.c_void_p), ("nQ", C.c_int), ("H", C.c_void_p),
                ("nH", C.c_int), ("c", C.c_void_p), ("nc", C.c_int), ("R", C.c_void_p),
                ("nR", C.c_int), ("mask", C.c_void_p)]


class FilterResult(C.Structure):
    _fields_ = [("pred_mean", C.c_void_p), ("pred_cov", C.c_void_p), ("filt_mean", C.c_void_p),
                ("filt_cov", C.c_void_p), ("log_marginal", C.c_void_p)]


class Noise(C.Structure):
    _fields_ = [("kind", C.c_int), ("keys", C.c_void_p), ("terminal", C.c_void_p),
                ("backward", C.c_void_p), ("bridge", C.c_void_p), ("n_bridge", C.c_longlong)]


class Target(C.Structure):
    _fields_ = [("kind", C.c_int), ("T", C.c_int), ("dx", C.c_int), ("ydim", C.c_int),
                ("linear", C.c_int), ("m0", C.c_void_p), ("P0", C.c_void_p), ("F", C.c_void_p),
                ("b", C.c_void_p), ("Q", C.c_void_p), ("nF", C.c_int), ("q", C.c_int),
                ("ne", C.c_int), ("exact_tv", C.c_int), ("eH", C.c_void_p), ("ec", C.c_void_p), ("eR", C.c_void_p),
                ("ey", C.c_void_p), ("emask", C.c_void_p), ("data", C.c_void_p),
                ("gmask", C.c_void_p), ("gH", C.c_void_p), ("gc", C.c_void_p),
                ("gR", C.c_void_p), ("lz_sigma", C.c_double), ("lz_rho", C.c_double),
                ("lz_beta", C.c_double), ("lz_h", C.c_double), ("l96_F", C.c_double),
                ("l96_h", C.c_double), ("exact_sel", C.c_int)]


class KernelOptions(C.Structure):
    _fields_ = [("backend", C.c_int), ("parallel_filter", C.c_int), ("zeroth_order", C.c_int)]


class KernelStats(C.Structure):
    _fields_ = [("accepted", C.c_longlong), ("rejected", C.c_longlong),
                ("aborted", C.c_longlong), ("nonfinite_gamma", C.c_longlong),
                ("last_log_alpha", C.c_double), ("last_accept_prob", C.c_double)]


class Chains(C.Structure):
    _fields_ = [("C", C.c_int), ("x", C.c_void_p), ("delta", C.c_void_p),
                ("log_gamma", C.c_void_p), ("grad_gen", C.c_void_p), ("iter", C.c_void_p),
                ("stats", C.c_void_p), ("root_keys", C.c_void_p)]


class PgChains(C.Structure):
    _fields_ = [("C", C.c_int), ("N", C.c_int), ("x", C.c_void_p), ("keys", C.c_void_p),
                ("delta", C.c_void_p), ("iter", C.c_void_p), ("updates", C.c_void_p),
                ("last_update", C.c_void_p), ("root_keys", C.c_void_p), ("status", C.c_void_p),
                ("bad_t", C.c_void_p), ("ancestors", C.c_void_p), ("selected", C.c_void_p),
                ("pm_kind", C.c_int)]


class ModelSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("T", C.c_int), ("dx", C.c_int), ("dy", C.c_int),
                ("grid", C.c_int), ("data_seed", C.c_uint64)] + [
        (n, C.c_double) for n in (
            "sv_mu sv_phi sv_sig2 sv_rho lz_sigma lz_rho lz_beta lz_h lz_gamma lz_obs_var "
            "st_phi st_kappa2 st_tau2 g1_phi g1_q g1_m0 g1_p0 l96_F l96_h l96_gamma "
            "l96_obs_var").split()]


VP = C.c_void_p
SIGNATURES = {
    "auxmc_version": (C.c_char_p, []),
    "auxmc_status_string": (C.c_char_p, [C.c_int]),
    "auxmc_device_ok": (C.c_int, []),
    "auxmc_last_error": (C.c_char_p, []),
    "auxmc_launch_count": (C.c_ulonglong, []),
    "auxmc_profile_begin": (None, []),
    "auxmc_profile_end": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]),
    "auxmc_rng_from_seed": (C.c_uint64, [C.c_uint64]),
    "auxmc_rng_derive": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "auxmc_rng_uniform": (C.c_double, [C.c_uint64, C.c_uint64]),
    "auxmc_rng_normal": (C.c_double, [C.c_uint64, C.c_uint64]),
    "auxmc_rng_normals": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int, VP,
                                    VP]),
    "auxmc_kalman_filter": (C.c_int, [C.POINTER(Lgssm), VP, C.c_int, C.c_int,
                                      C.POINTER(FilterResult), VP, VP, C.c_size_t, VP]),
    "auxmc_kalman_filter_workspace": (C.c_size_t, [C.POINTER(Lgssm), C.c_int, C.c_int]),
    "auxmc_dnc_bridge_count": (C.c_longlong, [C.c_int]),
    "auxmc_tshard_geometry": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    "auxmc_tshard_filter_workspace": (C.c_size_t, [C.POINTER(Lgssm)]),
    "auxmc_tshard_filter_local": (C.c_int, [C.POINTER(Lgssm), VP, C.c_int, C.c_int, VP,
                                            C.c_size_t, VP, VP, VP]),
    "auxmc_tshard_filter_finish": (C.c_int, [C.POINTER(Lgssm), VP, C.c_int, C.c_int, VP,
                                             C.c_size_t, VP, C.POINTER(FilterResult), VP, VP,
                                             VP]),
    "auxmc_tshard_sum": (C.c_int, [VP, C.c_int, VP, VP]),
    "auxmc_tshard_prefix_geometry": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "auxmc_tshard_prefix_workspace": (C.c_size_t, [C.POINTER(Lgssm)]),
    "auxmc_tshard_prefix_local": (C.c_int, [C.POINTER(Lgssm), C.POINTER(FilterResult),
                                            C.POINTER(Noise), C.c_int, C.c_int, VP, C.c_size_t,
                                            VP, VP, VP, VP, VP]),
    "auxmc_tshard_prefix_finish": (C.c_int, [C.POINTER(Lgssm), C.POINTER(Noise), C.c_int,
                                             C.c_int, VP, C.c_size_t, VP, VP, VP, VP]),
    "auxmc_sample_paths": (C.c_int, [C.POINTER(Lgssm), C.POINTER(FilterResult), C.c_int,
                                     C.POINTER(Noise), C.c_int, C.c_int, VP, VP, VP, C.c_size_t,
                                     VP]),
    "auxmc_sample_paths_workspace": (C.c_size_t, [C.POINTER(Lgssm), C.c_int, C.c_int, C.c_int]),
    "auxmc_sample_paths_host": (C.c_int, [C.POINTER(Lgssm), C.POINTER(FilterResult), C.c_int,
                                          VP, C.c_int, C.c_int, VP, VP]),
    "auxmc_rts_smoother": (C.c_int, [C.POINTER(Lgssm), C.POINTER(FilterResult), C.c_int, VP, VP,
                                     VP, VP, C.c_size_t, VP]),
    "auxmc_rts_smoother_workspace": (C.c_size_t, [C.POINTER(Lgssm), C.c_int]),
    "auxmc_affine_law": (C.c_int, [C.POINTER(Lgssm), C.POINTER(FilterResult), C.c_int, VP, VP,
                                   VP, VP, C.c_size_t, VP]),
    "auxmc_affine_law_workspace": (C.c_size_t, [C.POINTER(Lgssm), C.c_int]),
    "auxmc_test_flip_backward_gain": (C.c_int, [C.c_int]),
    "auxmc_test_force_generic_filter": (C.c_int, [C.c_int]),
    "auxmc_test_capture_log_marginal": (C.c_int, [C.c_void_p]),
    "auxmc_test_pfg_fixed_point": (C.c_int, [C.c_int]),
    "auxmc_test_pfg_fixed_point_steps": (C.c_longlong, [C.c_int]),
    "auxmc_path_logpdf": (C.c_int, [C.POINTER(Lgssm), VP, C.c_int, VP, C.POINTER(FilterResult),
                                    C.c_int, C.c_int, VP, VP, VP]),
    "auxmc_init_chains": (C.c_int, [C.POINTER(Target), C.POINTER(Chains), VP, C.c_size_t, VP]),
    "auxmc_aux_kernel_step": (C.c_int, [C.POINTER(Target), C.POINTER(Chains),
                                        C.POINTER(KernelOptions), VP, C.c_size_t, VP]),
    "auxmc_aux_kernel_workspace": (C.c_size_t, [C.POINTER(Target), C.c_int,
                                                C.POINTER(KernelOptions)]),
    "auxmc_adapt_delta": (C.c_int, [C.POINTER(Chains), C.c_double, VP]),
    "auxmc_gamma_move": (C.c_int, [C.POINTER(Target), C.c_int, VP, VP, C.c_longlong, C.c_double,
                                  VP, VP, VP]),
    "auxmc_tshard_aux_workspace": (C.c_size_t, [C.POINTER(Target)]),
    "auxmc_tshard_aux_begin": (C.c_int, [C.POINTER(Target), C.POINTER(Chains),
                                         C.POINTER(KernelOptions), VP, C.c_size_t, C.c_int,
                                         C.c_int, C.POINTER(Lgssm), C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), VP]),
    "auxmc_tshard_aux_middle": (C.c_int, [C.POINTER(Target), C.POINTER(Chains),
                                          C.POINTER(KernelOptions), VP, C.c_size_t, C.c_int,
                                          C.c_int, VP, VP, VP]),
    "auxmc_tshard_aux_end": (C.c_int, [C.POINTER(Target), C.POINTER(Chains),
                                       C.POINTER(KernelOptions), VP, C.c_size_t, C.c_int, C.c_int,
                                       VP, VP, VP]),
    "auxmc_tshard_aux_decide": (C.c_int, [C.POINTER(Target), C.POINTER(Chains), VP, C.c_size_t,
                                          C.c_int, C.c_int, VP, C.c_int, VP, VP, VP, VP]),
    "auxmc_copy_device": (C.c_int, [VP, VP, C.c_size_t, VP]),
    "auxmc_log_gamma": (C.c_int, [C.POINTER(Target), VP, C.c_int, VP, VP, VP]),
    "auxmc_aux_pgibbs_step": (C.c_int, [C.POINTER(Target), C.POINTER(PgChains), C.c_int,
                                        C.c_int, VP, C.c_size_t, VP]),
    "auxmc_aux_pgibbs_workspace": (C.c_size_t, [C.POINTER(Target), C.c_int, C.c_int, C.c_int]),
    "auxmc_pg_adapt_delta": (C.c_int, [C.POINTER(PgChains), C.c_double, VP]),
    "auxmc_spec_default": (None, [C.POINTER(ModelSpec)]),
    "auxmc_latent_dim": (C.c_int, [C.POINTER(ModelSpec)]),
    "auxmc_obs_dim": (C.c_int, [C.POINTER(ModelSpec)]),
    "auxmc_simulate": (C.c_int, [C.POINTER(ModelSpec), PD, PD]),
    "auxmc_synth_mats": (C.c_int, [C.POINTER(ModelSpec), PD, PD, PD, PD, PD, PD, PD]),
    "auxmc_target_params": (C.c_int, [C.POINTER(ModelSpec), PD, PD, PD, PD, PD]),
}

_lib = None


def load(require: bool = True):
    """Load libauxmc_b200.so; raises if absent (there is no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            if not require:
                return None
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2303_00301_b200.build` "
                "(the B200 path has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class AuxmcError(RuntimeError):
    def __init__(self, code: int, what: str):
        lib = load()
        msg = lib.auxmc_status_string(code).decode()
        extra = lib.auxmc_last_error().decode() if code == E_CUDA else ""
        super().__init__(f"{what}: {msg} ({code}) {extra}".strip())
        self.code = code


def check(code: int, what: str):
    if code != OK:
        raise AuxmcError(code, what)
