"""The CUDA kernel's 3x3 SoS epsilon order (extract3d.cu cPP3, a literal table) against two derivations
that share nothing with it: the Leibniz expansion of det(M + E) (tools/derive_sos3.py) and the oracle's
own order (ftko_sos_order: partial permutations sorted by exponent).  DESIGN.md reading R4."""
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def kernel_table():
    src = open(os.path.join(ROOT, "paper_2011_08697_b200", "csrc", "extract3d.cu")).read()
    m = re.search(r"__constant__ PP3 cPP3 = \{34, \{(.*?)\}\};", src, re.S)
    assert m
    rows = re.findall(r"\{(-?\d+), (-?\d+), (-?\d+)\}", m.group(1))
    return [tuple(int(v) for v in r) for r in rows]


def test_kernel_table_is_the_leibniz_order():
    import derive_sos3
    assert kernel_table() == derive_sos3.derive(3)


def test_kernel_table_is_the_oracle_order(oracle_lib):
    order = oracle_lib.sos_order(3)  # [k, 3]: perturbed column per row, -1 none
    assert [tuple(int(c) for c in row) for row in order] == kernel_table()
