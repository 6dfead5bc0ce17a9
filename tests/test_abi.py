"""CPU: the C-ABI library loads and exports every symbol include/enkf_mc.h declares; the product
package never touches the oracle; compute entry points fail loudly without a GPU."""

import ast
import os
import re

import numpy as np
import pytest

import paper_1606_00807_b200 as mck
from paper_1606_00807_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "enkf_mc.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(enkfmc_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.lib()
    declared = _declared()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.SYMBOLS) == declared
    assert b"sm_100a" in lib.enkfmc_version()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1606_00807_b200")
    for fn in os.listdir(pkg):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, fn)).read())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            assert not any(n.split(".")[0] == "oracle" for n in names), fn


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    geo = mck.GridGeometry("grid2d", 4, 4)
    X = np.random.default_rng(0).standard_normal((16, 6))
    net = mck.ObservationNetwork(np.array([1, 5]), np.array([0.1, 0.1]), np.zeros(2))
    with pytest.raises(mck.BackendError):
        mck.assimilate_parallel(mck.EnsembleState(X), net, mck.AssimilationConfig(zeta=1, delta=4), geo, Ys=np.zeros((2, 6)))
    with pytest.raises(mck.BackendError):
        mck.center_rows(X)
    with pytest.raises(mck.BackendError):
        mck.regression_solve(X[:3], X[4])
