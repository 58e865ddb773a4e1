"""ResNet-50's executable graph (paper_1901_05803_b200/resnet.py) against the catalog: every
linearised entry's parameters, output elements and FLOPs re-derived from the architecture, the
block-granularity lowering, the split mapping, the synthetic parameters, and the oracle's byte count
for the layer-placed and all-on-PS steps (CPU only)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import resnet, synthetic
from paper_1901_05803_b200.executor import ExecutorError, block_param_counts, lower
from paper_1901_05803_b200.planner import catalog_lookup, profile, volume_baseline, volume_ralp

REF = Path("/root/reference/pkg/src")


def test_geometry_matches_the_mirror_catalog():
    m = catalog_lookup("resnet-50")
    resnet.check_catalog(m)
    assert sum(L.param_count for L in m.layers) == 25_557_032   # pkg/tests/test_catalog.py:23-32


def test_geometry_matches_the_reference_catalog():
    if not (REF / "ralp" / "__init__.py").exists():
        pytest.skip("the reference package is not present on this machine")
    sys.path.insert(0, str(REF))
    try:
        import ralp
    finally:
        sys.path.remove(str(REF))
    ref = ralp.catalog_lookup("resnet-50")
    resnet.check_catalog(ref)
    ours = catalog_lookup("resnet-50")
    for b in (32, 64, 128):
        assert profile(ours.with_batch_size(b)).split_index == ralp.profile(ref.with_batch_size(b)).split_index


def test_lowering_and_split_mapping():
    layers = lower(catalog_lookup("resnet-50"))
    kinds = [L["kind"] for L in layers]
    assert kinds == ["conv", "pool"] + ["block"] * 16 + ["apool", "fc"]
    assert sum(L.get("downsample", 0) for L in layers) == 4
    assert [L["stride"] for L in layers if L["kind"] == "block" and L["downsample"]] == [1, 2, 2, 2]
    assert resnet.lowered_split(55) == 19 and resnet.lowered_split(2) == 2 and resnet.lowered_split(6) == 3
    with pytest.raises(ValueError):
        resnet.lowered_split(4)   # inside block s1b1
    params = synthetic.init_params(layers, 0)
    total = sum(p[0].size + p[1].size for p in params if p is not None)
    assert total == 25_557_032
    for L, p in zip(layers, params):
        if L["kind"] == "block":
            assert (p[0].size, p[1].size) == block_param_counts(L)


@pytest.mark.parametrize("split", [55, 2])
def test_oracle_bytes_are_the_cost_model(split):
    m = catalog_lookup("resnet-50").with_batch_size(2)
    layers = lower(m)
    st = ostep.OracleState(layers, synthetic.init_params(layers, 0))
    batches = [synthetic.batch(0, 0, r * 2, 2, (224, 224, 3), 1000) for r in range(2)]
    _, wire = ostep.train_step(st, "ralp", 2, batches, lr=1e-3, split=resnet.lowered_split(split))
    assert wire == volume_ralp(m, split, 2).total_bytes_per_step
    st = ostep.OracleState(layers, synthetic.init_params(layers, 0))
    _, wire = ostep.train_step(st, "baseline", 2, batches, lr=1e-3)
    assert wire == volume_baseline(m, 2).total_bytes_per_step
