"""A few 2-D efficiency-model iterations on 16384^2 (target for ncu captures of eff_round_*)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_cs_0502039_b200 as aca  # noqa: E402

aca.aca_efficiency_run((16384, 16384), 4, law=0, seed=5)
