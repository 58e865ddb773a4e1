"""Planner behaviour tests mirroring the reference's own test strategy
(pkg/tests/test_layers.py, test_descriptor.py, test_profiler.py, test_costmodel.py):
counting rules, descriptor errors, gate semantics, strategy validation, properties."""
import random
import warnings

import pytest

from oracle import planner as oplan
from paper_1901_05803_b200 import planner as P


def test_counting_rules():
    params, shape, flops = P.infer_conv(P.TensorShape(224, 224, 3), 3, 64, pad=1)
    assert params == 3 * 3 * 3 * 64 + 64 and (shape.h, shape.w, shape.c) == (224, 224, 64)
    assert flops == 2 * 9 * 3 * 64 * 224 * 224
    assert P.infer_pool(P.TensorShape(224, 224, 64), 2)[1] == P.TensorShape(112, 112, 64)
    assert P.infer_pool(P.TensorShape(55, 55, 64), 3, 2)[1] == P.TensorShape(27, 27, 64)
    assert P.infer_fc(25088, 4096) == (25088 * 4096 + 4096, P.TensorShape.flat(4096), 2 * 25088 * 4096)
    assert P.conv_output_hw(227, 227, 11, 4, 0) == (55, 55)
    assert P.TensorShape(7, 7, 512).elems == 25088 and str(P.TensorShape.flat(9)) == "9"
    with pytest.raises(P.ModelError):
        P.conv_output_hw(2, 2, 5, 1, 0)
    with pytest.raises(P.ModelError):
        P.infer_conv(P.TensorShape.flat(10), 3, 4)
    assert oplan.conv_counts(3, 64, 64, 224, 224) == (36928, 2 * 9 * 64 * 64 * 224 * 224)
    assert oplan.fc_counts(4096, 1000) == (4097000, 2 * 4096 * 1000)


def test_layerspec_and_graph_validation():
    with pytest.raises(P.ModelError):
        P.LayerSpec(index=0, name="x", kind=P.LayerKind.FULLY_CONNECTED, param_count=1,
                    output_elems_per_sample=1, compute_flops_per_sample=1)
    with pytest.raises(P.ModelError):
        P.LayerSpec(index=1, name="p", kind=P.LayerKind.POOLING, param_count=5,
                    output_elems_per_sample=1, compute_flops_per_sample=0)
    with pytest.raises(P.ModelError):
        P.LayerSpec(index=1, name="p", kind=P.LayerKind.POOLING, param_count=0,
                    output_elems_per_sample=0, compute_flops_per_sample=0)
    l1 = P.LayerSpec(index=2, name="a", kind=P.LayerKind.FULLY_CONNECTED, param_count=1,
                     output_elems_per_sample=1, compute_flops_per_sample=1)
    with pytest.raises(P.ModelError):
        P.ModelGraph("m", (l1,), 1)
    with pytest.raises(TypeError):
        l1.hyperparams["k"] = 3  # frozen mapping


def test_descriptor_errors_and_shape_checks():
    with pytest.raises(P.DescriptorError):
        P.parse_model("")
    with pytest.raises(P.DescriptorError):
        P.parse_model("conv1 conv k=3 cout=4")
    with pytest.raises(P.DescriptorError) as e:
        P.parse_model("model m batch=2 input=8x8x3\nc1 conv k=3 cout=x")
    assert e.value.line == 2
    with pytest.raises(P.ShapeMismatchError):
        P.parse_model("model m batch=2 input=8x8x3\nc1 conv k=3 cin=4 cout=8 pad=1")
    with pytest.raises(P.ShapeMismatchError):
        P.parse_model("model m batch=2 input=8x8x3\nc1 conv k=3 cout=8 pad=1\nf fc in=10 out=3")
    with pytest.raises(P.DescriptorError):
        P.parse_model("model m batch=2 input=8x8x3\nb1 block k=3")
    with pytest.raises(P.DescriptorError):
        P.parse_model("model m batch=2\nc1 conv k=3 cout=8")
    with pytest.raises(P.DescriptorError):
        P.parse_model("model m batch=2 input=8x8x3\nc1 wat k=3")
    g = P.parse_model("model m batch=2 elem_bytes=2 input=8x8x3 # comment\n"
                      "b1 block params=10 out=64 flops=5 shape=4x4x4\nf fc out=3\n")
    assert g.bytes_per_element == 2 and g.layer(2).param_count == 64 * 3 + 3


def test_gate_is_strict_and_threshold_warning():
    assert not P.gate_eligibility(-0.5, P.ProfilerConfig())
    assert P.gate_eligibility(-0.5000001, P.ProfilerConfig())
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        P.ProfilerConfig(threshold=0.1)
    assert w
    with pytest.raises(P.ProfilerError):
        P.compute_skewness([1])
    with pytest.raises(P.ProfilerError):
        P.compute_skewness([0, 0])
    with pytest.raises(P.ProfilerError):
        P.compute_skewness([1, -1])
    with pytest.raises(P.ProfilerError):
        P.gate_eligibility(float("nan"), P.ProfilerConfig())


def test_skewness_properties():
    rnd = random.Random(7)
    for _ in range(50):
        p = [rnd.randrange(1, 1000) for _ in range(rnd.randint(2, 30))]
        s = P.compute_skewness(p)
        assert abs(P.compute_skewness([x * 17 for x in p]) - s) < 1e-9          # scale invariance
        assert abs(P.compute_skewness(p[::-1]) + s) < 1e-9                     # reversal antisymmetry


def test_strategy_and_jobspec_validation():
    g = P.catalog_lookup("vgg16")
    with pytest.raises(P.CostModelError):
        P.Strategy(P.StrategyKind.RALP)
    with pytest.raises(P.CostModelError):
        P.Strategy(P.StrategyKind.BASELINE_PS, 3)
    with pytest.raises(P.CostModelError):
        P.JobSpec(g, P.Strategy.ralp(18), 2, ps_count=2)
    with pytest.raises(P.CostModelError):
        P.JobSpec(g, P.Strategy.ralp(21), 2)
    with pytest.raises(P.CostModelError):
        P.JobSpec(g, P.Strategy.ring(), 2, ps_count=1)
    with pytest.raises(P.CostModelError):
        P.JobSpec(g, P.Strategy.baseline(), 0)
    with pytest.raises(P.CostModelError):
        P.gpu_assignments(1)


def test_volume_properties():
    g = P.catalog_lookup("vgg16").with_batch_size(128)
    base = P.volume_ralp(g, 18, 1).total_bytes_per_step
    for w in (1, 2, 3, 8):
        v = P.volume_ralp(g, 18, w)
        assert v.total_bytes_per_step == w * base                                # linear in W
        assert v.parameter_sync_bytes + v.activation_bytes == v.total_bytes_per_step
    g2 = g.with_batch_size(256)
    assert (P.volume_ralp(g2, 18, 1).activation_bytes == 2 * P.volume_ralp(g, 18, 1).activation_bytes)
    # back-segment invariance: changing FC widths past the split never changes the volume
    text = P.serialize_model(g).replace("fc2 fc out=4096", "fc2 fc out=4096")
    assert P.volume_ralp(P.parse_model(text), 18, 4) == P.volume_ralp(g, 18, 4)


def test_catalog_override(tmp_path, monkeypatch):
    (tmp_path / "tiny.model").write_text("model tiny batch=4 input=8x8x3\nc conv k=3 cout=16 pad=1\n"
                                         "p pool window=2\nf fc out=10\n")
    monkeypatch.setenv(P.CATALOG_ENV_VAR, str(tmp_path))
    assert P.catalog_names() == ["tiny"]
    with pytest.raises(P.UnknownModelError):
        P.catalog_lookup("vgg16")
    assert P.catalog_lookup("tiny").num_layers == 3


def test_volume_ralp_multi_ps_extension():
    """The multi-PS extension: cut all-gather + cut-gradient reduce-scatter,
    row-parallel partials of the second FC layer to the PS and its gradient back, conv sync."""
    from paper_1901_05803_b200.planner import catalog_lookup, volume_ralp, volume_ralp_multi_ps
    m = catalog_lookup("vgg16").with_batch_size(128)
    for w in (1, 2, 4, 8):
        v = volume_ralp_multi_ps(m, 18, w)
        cut = m.output_bytes(18)
        fc2 = m.output_bytes(20)
        assert v.activation_bytes == 2 * w * (w - 1) * cut + 2 * (w - 1) * w * fc2
        assert v.parameter_sync_bytes == volume_ralp(m, 18, w).parameter_sync_bytes
        assert v.total_bytes_per_step == v.activation_bytes + v.parameter_sync_bytes
    assert volume_ralp_multi_ps(m, 18, 1).activation_bytes == 0
