"""paper_1312_3613_b200 -- B200-native data-parallel MCMC sweep (Augur, arXiv 1312.3613).

The product is libbnmc_gpu.so (C-ABI: include/bnmc_gpu.h), hand-written CUDA for
sm_100a.  This package holds its sources (csrc/), the in-tree build
(build.py) and a Python mirror of the reference sampler API (engine.py).
"""
from .engine import (BnmcError, CudaError, DomainError, Engine, ParamStore, RunConfig,  # noqa: F401
                     dirichlet_batch, layout_lengths, lib, log_predictive_probability, map_estimate,
                     nccl_unique_id, partition, PeerGroup, probe_gamma, probe_log_weights, probe_rng, read_bandwidth,
                     sample, write_corpus, lpp_curve)
