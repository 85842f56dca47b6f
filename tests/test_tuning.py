"""The drop-in constructor keeps the reference's signature plus one validated
``tuning`` mapping."""
import inspect

import pytest

from paper_1906_05737_b200 import CompiledNetwork, compile_model
from paper_1906_05737_b200.kernels import Specializer
from paper_1906_05737_b200.tuning import FIELDS, Tuning, make_tuning


def test_constructor_signature_is_reference_plus_four_keywords():
    params = inspect.signature(CompiledNetwork.__init__).parameters
    assert list(params) == ["self", "manifest", "weights", "options", "batch", "device",
                            "cache_dir", "tuning"]


def test_unknown_key_raises_value_error_naming_the_valid_keys():
    with pytest.raises(ValueError, match="unknown tuning key.*tc_min_rowz.*valid keys: gpu_fusion"):
        make_tuning({"tc_min_rowz": 1})
    with pytest.raises(ValueError, match="mapping"):
        make_tuning(42)


def test_defaults_and_overrides():
    assert make_tuning(None) == Tuning()
    t = make_tuning({"tc_min_rows": 1, "dw_fusion": False})
    assert t.tc_min_rows == 1 and t.dw_fusion is False and t.use_tc
    assert make_tuning(t) is t


def test_every_specializer_knob_is_a_tuning_field():
    spec = set(inspect.signature(Specializer.__init__).parameters) - {
        "self", "plan", "assignment", "options", "max_batch", "capacity", "sm_count"}
    kw = Tuning().specializer_kwargs()
    assert set(kw) == spec, set(kw) ^ spec
    assert set(FIELDS) == spec | {"gpu_fusion", "dw_fusion", "chain", "tc_chain", "pw_dw", "gap_dense"}
    assert kw["tc_min_rows"] == 256 and make_tuning({"mega": True}).specializer_kwargs()[
        "tc_min_rows"] == 2048


def test_compile_model_rejects_stray_keywords_before_any_gpu_work():
    from paper_1906_05737_b200 import zoo
    m, w = zoo.build(0)
    with pytest.raises(TypeError):
        compile_model(m, w, None, batch=4, tc_min_rows=1)
