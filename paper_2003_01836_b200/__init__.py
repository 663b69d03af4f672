"""B200-native (sm_100a) barycentric Lagrange treecode evaluation path.

Drop-in for the reference package's evaluation entry points
(``bltc.engine.treecode_potentials``, ``bltc.decomp.run_distributed``);
all compute runs in libbltc.so (csrc/, C ABI in include/bltc.h).
"""
from .engine import (Context, EvalConfig, RunStats, cheb_nodes, default_context,
                     treecode_potentials)
from .kernels import KernelKind, KernelSpec, coulomb, eval_kernel, test_constant, yukawa
from .particles import ParticleSystem, Points, read_particles_csv, write_particles_csv

__all__ = [
    "Context", "EvalConfig", "RunStats", "cheb_nodes", "default_context",
    "treecode_potentials", "KernelKind", "KernelSpec", "coulomb", "eval_kernel",
    "test_constant", "yukawa", "ParticleSystem", "Points", "read_particles_csv",
    "write_particles_csv",
]
