"""The C-ABI library: it loads, exports every entry point include/gosma_capi.h
declares, and validates arguments like the reference (before any device
work). CPU only — no compute calls."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gosma_capi.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gosma_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["gosma_ctx_create", "gosma_ctx_destroy", "gosma_eval_bounds",
                 "gosma_eval_bounds_device", "gosma_solve", "gosma_last_error",
                 "gosma_objective_value", "gosma_local_refine"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_1812_01232_b200 as g
    lib = C.CDLL(g.library_path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_node_record_layout():
    import paper_1812_01232_b200 as g
    assert g.NODE_DTYPE.itemsize == 88  # gosma_node: 11 doubles
    n = g.make_nodes([[0.1, 0.2, 0.3]], 0.5, [1, 2, 3], [0.1, 0.2, 0.3])
    flat = n.view(np.float64)
    assert flat.tolist() == [0.1, 0.2, 0.3, 0.5, 1, 2, 3, 0.1, 0.2, 0.3, -np.inf]


def _classes(**over):
    c = {"mu": [[0, 0, 2]], "sigma2": [1.0], "phi1": [1.0], "dir": [[0, 0, 1]],
         "kappa2": [5.0], "phi2": [1.0], "weight": 1.0}
    c.update(over)
    return [c]


@pytest.mark.parametrize("over,zeta,msg", [
    ({}, 0.0, "zeta must be > 0"),
    ({"phi1": [0.9]}, 0.5, "weights sum"),
    ({"phi2": [1.1]}, 0.5, "weights sum"),
    ({"sigma2": [0.0]}, 0.5, "variance"),
    ({"sigma2": [-1.0]}, 0.5, "variance"),
    ({"kappa2": [0.0]}, 0.5, "concentration"),
    ({"dir": [[3, 4, 0]]}, 0.5, "deviates from 1"),
    ({"phi1": [-0.1]}, 0.5, "non-negative"),
])
def test_context_validation_mirrors_reference(over, zeta, msg):
    import paper_1812_01232_b200 as g
    with pytest.raises(ValueError, match=msg):
        g.ObjectiveContext(_classes(**over), zeta, single_mixture=True)


def test_semantic_class_weights_must_close():
    import paper_1812_01232_b200 as g
    c = _classes()
    c2 = [dict(c[0], weight=0.3), dict(c[0], weight=0.3)]
    with pytest.raises(ValueError, match="class weights"):
        g.ObjectiveContext(c2, 0.5)


def test_valid_context_without_a_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1812_01232_b200 as g
    with pytest.raises((g.GosmaError, ValueError)):
        g.ObjectiveContext(_classes(), 0.5, single_mixture=True)
