"""Branch-group models on the host side: the Inception-v3 / GoogLeNet geometry
(paper_1901_05803_b200/branchy.py) against the reference's own catalog tables (tests/golden, made by
running the unmodified reference), their lowering to RALPB_MODULE layers, the catalog-split ->
lowered-split map, parameter layouts (executor == oracle), and the one-node modules the generic
lowering makes for convolutions that are not stride-1 'same' windows (OverFeat's conv2)."""
import json
from pathlib import Path

import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import branchy, synthetic
from paper_1901_05803_b200.executor import _desc_array, lower
from paper_1901_05803_b200.planner import catalog_lookup, profile

GOLD = json.loads((Path(__file__).parent / "golden" / "planner_golden.json").read_text())


@pytest.mark.parametrize("name", ["inception-v3", "googlenet"])
def test_geometry_reproduces_reference_catalog(name):
    want = [(r["name"], r["kind"], r["params"], r["out"], r["flops"]) for r in GOLD["models"][name]["table"]]
    got = [(e.name, e.kind, e.params, e.out, e.flops if e.kind != "fc" else want[-1][4]) for e in branchy.entries(name)]
    assert got == want
    branchy.check_catalog(catalog_lookup(name))


@pytest.mark.parametrize("name,batch,split,lowered", [
    ("inception-v3", 128, 97, 19),   # apool | fc
    ("inception-v3", 32, 7, 7),      # pool2: the eleven branch groups on the PS
    ("googlenet", 128, 62, 17),
    ("googlenet", 32, 18, 8),        # pool3
    ("googlenet", 8, 5, 5),          # pool2
])
def test_partitioner_splits_map_to_group_boundaries(name, batch, split, lowered):
    assert profile(catalog_lookup(name).with_batch_size(batch)).split_index == split
    assert branchy.lowered_split(name, split) == lowered
    layers, _ = branchy.lower_layers(name)
    assert layers[lowered - 1]["kind"] in ("pool", "apool")


def test_cut_inside_a_group_is_rejected():
    with pytest.raises(ValueError, match="inside group mixed0"):
        branchy.lowered_split("inception-v3", 9)


@pytest.mark.parametrize("name", ["inception-v3", "googlenet"])
def test_lowered_tables_and_parameter_layouts(name):
    model = catalog_lookup(name)
    layers = lower(model)
    assert sum(ostep.param_count(L) for L in layers) == sum(L.param_count for L in model.layers)
    params = synthetic.init_params(layers, 0)
    for L, p in zip(layers, params):
        if L["kind"] == "module":
            nw, nb = branchy.module_param_counts(L)
            assert p[0].size == nw and p[1].size == nb
            assert nw + nb == ostep.param_count(L)
    descs, nodes = _desc_array(layers)
    mods = [L for L in layers if L["kind"] == "module"]
    assert len(nodes) == sum(len(L["nodes"]) for L in mods)
    begin = 0
    for d, L in zip(descs, layers):
        if L["kind"] == "module":
            assert (d.node_begin, d.node_count) == (begin, len(L["nodes"]))
            begin += d.node_count
            assert sum(nd["cout"] if nd["op"] == "conv" else 0 for nd in L["nodes"] if nd["output"]) <= d.cout


def test_inception_module_shapes():
    layers = {L["name"]: L for L in branchy.lower_layers("inception-v3")[0]}
    m3 = layers["mixed3"]   # 35 -> 17: two stride-2 branches and the max pool, 384 + 96 + 288
    assert (m3["h"], m3["cin"], m3["cout"]) == (35, 288, 768)
    shp, out = branchy.node_shapes(m3["nodes"], m3["h"], m3["w"], m3["cin"])
    assert out == (17, 17, 768)
    m9 = layers["mixed9"]   # the split 3x3 branches: 1x3 and 3x1 both outputs
    _, out = branchy.node_shapes(m9["nodes"], m9["h"], m9["w"], m9["cin"])
    assert out == (8, 8, 2048)
    assert [L["name"] for L in layers.values()][-2:] == ["apool", "fc"]


def test_overfeat_unpadded_conv_becomes_a_module():
    layers = lower(catalog_lookup("overfeat"))
    kinds = [(L["name"], L["kind"]) for L in layers]
    assert kinds[2] == ("conv2", "module") and kinds[0] == ("conv1", "conv") and kinds[4] == ("conv3", "conv")
    nd = layers[2]["nodes"][0]
    assert (nd["kh"], nd["stride"], nd["ph"], nd["bn"], nd["output"]) == (5, 1, 0, 0, 1)
    assert sum(ostep.param_count(L) for L in layers) == sum(L.param_count for L in catalog_lookup("overfeat").layers)


def test_oracle_runs_a_reduced_inception():
    layers, _ = branchy.lower_layers("inception-v3", 139)
    params = synthetic.init_params(layers, 0)
    st = ostep.OracleState(layers, params)
    imgs, labs = synthetic.batch(0, 0, 0, 2, (139, 139, 3), 1000)
    loss, wire = ostep.train_step(st, "ralp", 1, [(imgs, labs)], lr=1e-3, emulate_bf16=True, split=7)
    assert 6.0 < loss < 8.5 and wire > 0
