"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds no arithmetic of the method (no rounding, no QR, no ID):
it only draws matrices A_D with the structure of the paper's workloads
(prescribed singular-value decay, P:207 and Table 3) and of
BASELINE.json's five configs.  See DESIGN.md "Input recipe".
"""
from .generators import (  # noqa: F401
    CONFIGS, ConfigSpec, config_spec, gen_config, gen_decay, gen_planted,
    gen_exact_rank, gen_fourier, fourier_params, haar, counter_normal, counter_sign, SKETCH_STREAM,
)
