"""B200-native KADABRA sampling hot path (arXiv 1910.11039), behind the reference library's entry points.

C ABI: include/ebc_b200.h -> paper_1910_11039_b200/libebc_b200.so (hand-written sm_100a CUDA).
This package is the thin host-side mirror used by tests and bench.py.
"""
from .api import (EMPIRICAL_BERNSTEIN, HOEFFDING, TAG_ADAPTIVE, TAG_CALIBRATION, UNIFORM, WEIGHTED,
                  WORK_NAMES, ApproxResult, BackendFault, ConfigError, CudaError, Graph, ParseError,
                  RunConfig, Sampler, algorithmic_bytes, calibrate, compute_omega, diameter_upper_bound,
                  epoch_length, gen_erdos_renyi, gen_grid, gen_rmat, gen_rmat_device, parse_allocator_kind,
                  parse_bound_kind, read_scores, release_device_cache, run_pipeline, shard_range, write_scores,
                  compare_score_files)
from .build import build

__all__ = [n for n in dir() if not n.startswith("_")]
