"""Seeded synthetic inputs for the LAKER hot path (shared by the CUDA path's
tests/bench and by the oracle's tests).

This package holds NO arithmetic of the method (no kernel, no PCG, no CCCP):
only the input recipe of DESIGN.md §3 (sensor locations, transmitters, RSS
values, embeddings, random directions).  See `synth.radio`.
"""
from .radio import (CONFIGS, ConfigSpec, Problem, make_problem, make_paper_problem, make_directions,
                    embed, grid_points, worked_example)

__all__ = ["CONFIGS", "ConfigSpec", "Problem", "make_problem", "make_paper_problem", "make_directions",
           "embed", "grid_points", "worked_example"]
