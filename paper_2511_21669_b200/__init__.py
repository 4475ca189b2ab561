"""B200-native DSD-Sim replica engine (arxiv 2511.21669 simulate-a-sweep path).

The product is libdsdsim.so (include/dsdsim.h): host C++ config/sweep/report
layer + sm_100a CUDA kernels.  This package is the thin Python mirror used by
tests and bench.py; see DESIGN.md.
"""
from .api import (ConfigError, DsdError, EngineError, SimulationOutput, Simulator, SweepOutput, SUMMARY_DTYPE,
                  build_scenarios, run_simulation, run_sweep, sweep_point_seed)

__all__ = ["ConfigError", "DsdError", "EngineError", "SimulationOutput", "Simulator", "SweepOutput",
           "SUMMARY_DTYPE", "build_scenarios", "run_simulation", "run_sweep", "sweep_point_seed"]
