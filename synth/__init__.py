"""Seeded synthetic inputs (circuits) shared by the oracle and the CUDA path.

Holds no arithmetic of the method (no op evaluation, no hashing, no stimulus
values): see DESIGN.md §"Inputs" for the recipe.
"""
from .circuit import Circuit, Builder, OP_NAMES, OP_BY_NAME, NUM_OPS  # noqa: F401
from .generator import CONFIGS, GenConfig, generate, config_circuit, fuzz_circuit, multicore_circuit  # noqa: F401
