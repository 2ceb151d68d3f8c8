"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no geometry factors, no
spectral factor, no operator).  It only draws the inputs the paper's
workloads are made of: a binary secondary mask, a Kramers source spectrum,
two-peak Gaussian momentum-transfer profiles painted into a phantom, and
Poisson counts.  See DESIGN.md "Input recipe".
"""
from .configs import CONFIGS, Config, make_config, poisson_data  # noqa: F401
