"""paper_2603_11340_b200 — the SLO-Tuner serving simulator (arXiv 2603.11340) as a batched Monte-Carlo
hot path on B200: C-ABI library libslosim.so (include/slo_sim.h) + a thin ctypes binding.

Submodules are imported lazily so that the seeded input generators (`inputs`) can be used without the
CUDA library; the simulation entry points (`sim`) raise if libslosim.so is missing — there is no CPU
fallback.
"""
import importlib

__all__ = ["inputs", "sim", "dist"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
