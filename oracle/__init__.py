"""TEST INFRASTRUCTURE ONLY: the CPU discrete-event oracle (see sf_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2601_12784_b200) never imports it.
"""
from .oracle import (OracleSim, Ledger, Params, InstView, TsItem, build_oracle,  # noqa: F401
                     load_oracle, oracle_config_from_preset, METRIC_NAMES)
