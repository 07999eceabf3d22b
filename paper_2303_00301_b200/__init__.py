"""B200-native hot path of auxmc 0.1.0 (arXiv 2303.00301): auxiliary Kalman and
auxiliary particle Gibbs samplers for state-space models.

Submodules mirror the reference namespaces: `rng` (rng.hpp), `lgssm`
(lgssm.hpp), `pit` (pit.hpp), `auxk` (auxk.hpp / target.hpp), `fkpg`
(fkpg.hpp), `bench_models` (bench/models.hpp).  All compute goes through
libauxmc_b200.so (include/auxmc_gpu.h); there is no CPU fallback.
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"


def library():
    return _lib.load()


def version() -> str:
    return _lib.load().auxmc_version().decode()
