"""CPU oracle (test infrastructure only; see ``oracle/sp_oracle.py`` header)."""
from .sp_oracle import *  # noqa: F401,F403
from .sp_oracle import (OracleConfig, SpatialPoolerOracle, StepResult, init_pools, encode,
                        overlap_raw, boost_integer, boost_overlap, inhibit, learn, sdr_words,
                        splitmix64_next, neighbourhood, TWO23)
