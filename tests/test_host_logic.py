"""CPU tests of the host-side logic around the kernels (no GPU calls)."""

import re
from pathlib import Path

import numpy as np
import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]


def test_greedy_order_matches_reference_rules():
    from paper_2409_14939_b200.trainer import greedy_order
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(2, 10))
        m = rng.choice([0.0, 0.25, 0.5, 1.0], size=(n, n)) if rng.random() < 0.5 else rng.random((n, n))
        m = np.triu(m, 1)
        m = m + m.T
        assert greedy_order(m) == oracle.greedy_order(m)


def test_counts_layout_matches_header():
    from paper_2409_14939_b200.sampler import counts_layout
    text = (ROOT / "include" / "fastgl_b200.h").read_text()
    macros = dict(re.findall(r"#define (FGL_CNT_\w+)\(H, nb\) (.*)", text))
    env = {}
    for H in (1, 2, 3, 5):
        for nb in (1, 2, 8):
            def ev(name):
                expr = macros[name].replace("(H)", str(H)).replace("(nb)", str(nb))
                for k in macros:
                    expr = expr.replace(f"{k}({H}, {nb})", str(env[k])) if k in env else expr
                return eval(re.sub(r"FGL_CNT_(\w+)\(H, nb\)", lambda mm: str(env["FGL_CNT_" + mm.group(1)]), expr))
            env.clear()
            for k in ("FGL_CNT_FRONT", "FGL_CNT_UNIQ", "FGL_CNT_DRAWS", "FGL_CNT_STATUS", "FGL_CNT_LEN"):
                env[k] = ev(k)
            lay = counts_layout(H, nb)
            assert lay["front"] == env["FGL_CNT_FRONT"] and lay["uniq"] == env["FGL_CNT_UNIQ"]
            assert lay["draws"] == env["FGL_CNT_DRAWS"] and lay["status"] == env["FGL_CNT_STATUS"]
            assert lay["len"] == env["FGL_CNT_LEN"]


def test_init_params_match_reference():
    from paper_2409_14939_b200.trainer import init_params
    for dims in ((16, 32, 2), (100, 64, 64, 47)):
        for (w, b), (w2, b2) in zip(init_params(dims, 3), oracle.init_params(dims, 3)):
            assert np.array_equal(w, w2) and np.array_equal(b, b2)


def test_model_config_validation():
    from paper_2409_14939_b200.errors import ValidationError
    from paper_2409_14939_b200.trainer import ModelConfig
    with pytest.raises(ValidationError):
        ModelConfig(layer_dims=(4, 2), fanouts=[2, 2])
    with pytest.raises(ValidationError):
        ModelConfig(layer_dims=(4, 2), fanouts=[2], arch="gat")
    with pytest.raises(ValidationError):
        ModelConfig(layer_dims=(4,), fanouts=[])
    with pytest.raises(ValidationError):
        ModelConfig(layer_dims=(4, 2), fanouts=[2], lr=-1.0)
    c = ModelConfig(layer_dims=(4, 3, 2), fanouts=[2, 1])
    assert c.num_layers == 2


def test_fanouts_validation():
    from paper_2409_14939_b200.errors import ValidationError
    from paper_2409_14939_b200.sampler import Fanouts
    assert list(Fanouts([3, 2])) == [3, 2]
    with pytest.raises(ValidationError):
        Fanouts([])
    with pytest.raises(ValidationError):
        Fanouts([1, 0])


def test_idmap_geometry_matches_reference():
    from paper_2409_14939_b200.idmap import _geometry
    for n in (1, 2, 3, 5, 1000, 1024, 1025, 10**6):
        assert _geometry(n, None, "fib") == oracle.minigl_oracle._table_geometry(n, None, "fib")
    assert _geometry(5, 8, "mod") == oracle.minigl_oracle._table_geometry(5, 8, "mod")


def test_shard_round_robin():
    from paper_2409_14939_b200.dist import shard
    items = list(range(11))
    parts = [shard(items, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == items
    assert parts[1] == [1, 5, 9]


def test_derive_seed_and_keys():
    from paper_2409_14939_b200.sampler import derive_seed, philox_key
    assert derive_seed(0, 13, 5) == oracle.derive_seed(0, 13, 5)
    assert philox_key(77) == oracle.philox.key_for_seed(77)
