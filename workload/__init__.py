"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and
bench.py: mechanism tables (read from data/mech/*.json), cell states shaped
like the paper's workloads (PAPER.md:222-231 H2 quasi-DNS/TGV, PAPER.md:263-267
CH4 LES), and random-init MLP bundles of the paper's shape.

This package holds NO arithmetic of the method (no NASA, transport, Box-Cox,
MLP or projection math); it only reads tables, draws random numbers and shapes
profiles.  Every value is a pure function of (SEED, field, global cell index),
so a shard of cells generated on its own equals the same cells of the whole.
"""
from .mech import load_kinetics, load_mech
from .cells import CONFIGS, make_cells, make_cells_at, tau_mix_at, Config
from .bundle import make_bundle

SEED = 231213513
__all__ = ["load_mech", "load_kinetics", "make_cells", "make_cells_at", "tau_mix_at", "make_bundle", "CONFIGS", "Config", "SEED"]
