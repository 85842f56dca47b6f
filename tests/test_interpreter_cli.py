"""The host-side SimpleNN analogue (interpret) and the CLI."""
import json
import subprocess
import sys

import numpy as np
import pytest

from builders import random_network
from golden_util import load, names
from oracle import oracle
from paper_1906_05737_b200 import build_graph, interpret, save_model, zoo
from paper_1906_05737_b200.cli import main

F32 = np.float32


@pytest.mark.parametrize("name", names())
def test_interpret_matches_reference_goldens_bit_exact(name):
    m, w, x, rec = load(name)
    g = build_graph(m, w)
    np.testing.assert_array_equal(interpret(g, [x], batched=True)[0], rec["interp"])
    np.testing.assert_array_equal(interpret(g, [x[0]])[0], rec["interp"][0])


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_interpret_matches_c_oracle_on_zoo(cfg):
    m, w = zoo.build(cfg)
    g = build_graph(m, w)
    x = zoo.inputs(cfg, 2)
    np.testing.assert_array_equal(interpret(g, [x], batched=True)[0],
                                  oracle.run_graph(g, [x])[0])


def test_interpret_random_networks():
    rng = np.random.default_rng(5)
    for _ in range(40):
        m, w, shape = random_network(rng)
        g = build_graph(m, w)
        x = rng.uniform(-2, 2, (2,) + shape).astype(F32)
        np.testing.assert_array_equal(interpret(g, [x], batched=True)[0],
                                      oracle.run_graph(g, [x])[0])


@pytest.fixture
def model_files(tmp_path):
    m, w, arrays = zoo.build(0, with_arrays=True)
    path = tmp_path / "cfg0.json"
    save_model(m, arrays, path)
    return str(path)


def test_inspect_text_and_json(model_files, capsys):
    assert main(["inspect", model_files]) == 0
    out = capsys.readouterr().out
    assert "units (5)" in out and "launches" in out and "+maxpool2" in out
    assert main(["inspect", model_files, "--json", "--batch", "4096", "--source"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert len(doc["units"]) == 5 and doc["capacity"] == 4096
    assert doc["source"].startswith('#include "nnb_kernels.cuh"')
    assert any("direct" in l["kernel"] for l in doc["launches"])


def test_usage_errors_exit_2(tmp_path, capsys):
    assert main(["inspect", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert main(["inspect", str(bad)]) == 2
    assert "error:" in capsys.readouterr().err


def test_closed_pipe_is_not_an_error(model_files):
    p = subprocess.run(f"{sys.executable} -m paper_1906_05737_b200 inspect {model_files} "
                       "--source | head -1", shell=True, capture_output=True, text=True,
                       cwd=str(__import__('pathlib').Path(__file__).resolve().parent.parent))
    assert p.returncode == 0 and p.stdout.startswith("units")
    assert "Traceback" not in p.stderr


@pytest.mark.gpu
def test_cli_verify_bench_run_on_gpu(model_files, tmp_path, capsys):
    assert main(["verify", model_files, "--mode", "exact", "--softmax-exp", "exact",
                 "--trials", "3", "--json"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["pass"] and rep["outputs"][0]["argmax_agree"]
    assert main(["verify", model_files, "--trials", "2", "--tol-abs", "0", "--json"]) == 1
    capsys.readouterr()
    assert main(["bench", model_files, "--runs", "5", "--warmup", "2", "--json",
                 "--batch", "64"]) == 0
    rep = json.loads(capsys.readouterr().out)
    for key in ("compile_ms", "mean_us", "std_us", "interpreter_mean_us", "speedup",
                "images_per_s", "gpu"):
        assert key in rep
    x = zoo.inputs(0, 1)[0]
    xp = tmp_path / "x.bin"
    xp.write_bytes(x.astype("<f4").tobytes())
    assert main(["run", model_files, str(xp), "--json", "--mode", "exact",
                 "--softmax-exp", "exact"]) == 0
    out = np.array(json.loads(capsys.readouterr().out)[0], F32)
    m, w = zoo.build(0)
    np.testing.assert_allclose(out, oracle.run(m, w, [x[None]])[0][0], rtol=1e-4, atol=1e-5)
    xp.write_bytes(b"123")
    assert main(["run", model_files, str(xp)]) == 2


@pytest.mark.gpu
def test_compiled_network_never_uses_host_compute(monkeypatch):
    """compile()/apply() run only the sm_100a kernels: break every host compute
    path and the network still produces oracle-exact results."""
    import paper_1906_05737_b200.interpreter as interp_mod

    def boom(*a, **k):
        raise AssertionError("host interpreter called on the product path")
    monkeypatch.setattr(interp_mod, "interpret", boom)
    monkeypatch.setattr(interp_mod, "_node", boom)
    from paper_1906_05737_b200 import EXACT, compile_model
    m, w = zoo.build(2)
    x = zoo.inputs(2, 3)
    net = compile_model(m, w, EXACT, batch=3)
    got = net.run([x])[0].cpu().numpy()
    np.testing.assert_allclose(got, oracle.run(m, w, [x])[0], rtol=1e-4, atol=1e-5)
