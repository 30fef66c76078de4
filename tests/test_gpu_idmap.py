"""GPU Fused-Map table vs the reference's golden table states (bit-exact keys,
values and slot layout) and its error contract."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_golden_traces(golden_meta):
    from paper_2409_14939_b200 import idmap
    for tr in golden_meta["idmap_traces"]:
        t = idmap.build(tr["ids"], capacity_override=tr["cap"], hash_kind=tr["kind"])
        assert t.capacity == tr["capacity"] and t.shift == tr["shift"]
        assert [int(k) for k in t.keys] == tr["keys"], tr
        assert [int(v) for v in t.values] == tr["values"], tr
        assert t.num_inserted == tr["num_inserted"]


def test_golden_layouts(golden):
    from paper_2409_14939_b200 import idmap
    st = golden("idmap")
    for name in ("rand_u62", "dups", "sorted", "bench_ids"):
        ids = st[f"{name}_ids"]
        t = idmap.build(ids, workers=8)
        assert np.array_equal(t.keys, st[f"{name}_keys"]), name
        assert np.array_equal(t.values, st[f"{name}_values"]), name
        got = idmap.lookup_many(t, ids)
        want = oracle.idmap_lookup(oracle.idmap_build(ids), ids)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("kind", ["fib", "mod"])
def test_random_layouts_vs_oracle(kind):
    from paper_2409_14939_b200 import idmap
    rng = np.random.default_rng(7)
    for trial in range(6):
        n = int(rng.integers(1, 3000))
        ids = rng.integers(0, int(rng.choice([50, 5000, 1 << 40])), size=n).astype(np.uint64)
        cap = None if kind == "fib" else int(rng.integers(len(np.unique(ids)), 3 * n + 2))
        t = idmap.build(ids, capacity_override=cap, hash_kind=kind)
        o = oracle.idmap_build(ids, capacity_override=cap, hash_kind=kind)
        assert np.array_equal(t.keys, o.keys) and np.array_equal(t.values, o.values)


def test_first_seen_and_errors():
    from paper_2409_14939_b200 import idmap
    from paper_2409_14939_b200.errors import CapacityError, NotFoundError, ValidationError
    t = idmap.build([50, 3, 99, 3, 12], workers=1)
    assert [idmap.lookup(t, g) for g in (50, 3, 99, 12)] == [0, 1, 2, 3]
    with pytest.raises(NotFoundError, match="7"):
        idmap.lookup(idmap.build([3]), 7)
    with pytest.raises(ValidationError):
        idmap.build([])
    with pytest.raises(ValidationError):
        idmap.build([int(idmap.SENTINEL)])
    with pytest.raises(ValidationError):
        idmap.build([1], capacity_override=6)  # fib needs a power of two
    with pytest.raises(CapacityError):
        idmap.build([1, 2, 3], capacity_override=2, hash_kind="mod")


def test_translate_batch_matches_oracle(powerlaw_10k):
    from paper_2409_14939_b200 import idmap, sampler
    b = sampler.sample_khop(powerlaw_10k, np.arange(0, 10_000, 97), [5, 3], 5)
    t = idmap.build(b.unique_nodes)
    tb = idmap.translate_batch(t, b)
    assert tb.num_local == len(b.unique_nodes)
    for (lt, ls, _), (gt, gs, _) in zip(tb.local_layers, b.layers):
        assert np.array_equal(lt, np.searchsorted(b.unique_nodes, gt))
        assert np.array_equal(ls, np.searchsorted(b.unique_nodes, gs))
