"""Write a small BTD1 container with the REAL reference's write_btd (build container only).

    python tests/golden/make_btd_golden.py    # needs /root/reference; writes tests/golden/ref_small.btd
"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import blocktri as bt  # noqa: E402

A, B = bt.generate_spd_btd(7, 3, 2, seed=5)
A.sub[2, 1, 1] = -0.0  # negative zero must round-trip bit-exactly
bt.write_btd(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_small.btd"), A, B)
