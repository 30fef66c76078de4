"""plan_tiles / TileConfig semantics (ConfigError before any compute) against
the reference's accept/reject table -- host-side validation, CPU only."""

import numpy as np
import pytest


def test_plan_tiles_table(golden_meta):
    from paper_2409_14939_b200 import compute
    from paper_2409_14939_b200.errors import ConfigError
    for p in golden_meta["plan_tiles"]:
        cfg = compute.TileConfig(p["x"], p["y"], p["scratch"])
        if p["ok"] is True:
            plan = compute.plan_tiles(p["nt"], p["d"], np.array(p["fanouts"], dtype=np.int64), cfg)
            assert plan.num_targets == p["nt"]
        else:
            with pytest.raises(ConfigError):
                compute.plan_tiles(p["nt"], p["d"], np.array(p["fanouts"], dtype=np.int64), cfg)


def test_plan_coverage():
    from paper_2409_14939_b200 import compute
    plan = compute.plan_tiles(37, 70, np.arange(37) % 5, compute.TileConfig(8, 32))
    cells = set()
    for t0, t1, c0, c1 in plan.tiles:
        cells |= {(t, c) for t in range(t0, t1) for c in range(c0, c1)}
    assert len(cells) == 37 * 70
