"""The C++ drop-in (include/rnntsim_cuda.hpp) run through the reference's own
acceptance checks in one binary (tests/cpp/test_dropin.cpp), built in the
build container by tests/cpp/Makefile (needs /root/reference headers) and
executed here on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_binary_built_or_buildable():
    if os.path.exists(BIN):
        return
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("drop-in binary not built and the reference headers are absent")
    subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "tests", "cpp", "Makefile")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_acceptance_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_dropin not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") >= 8


CLI = os.path.join(ROOT, "tools", "rnntg_cli")


@pytest.mark.gpu
@pytest.mark.parametrize("model,algo,extra", [
    ("neural:3", "graph", []),
    ("neural:3", "label_loop_graph", []),
    ("lstm:5", "graph", ["--layers", "2"]),
    ("lstm:5", "tdt_label_loop_graph", ["--layers", "2"]),
])
@pytest.mark.parametrize("exec_", ["tensor", "graph", "hostloop"])
def test_cli_decode_route_wer0(tmp_path, model, algo, extra, exec_):
    """The reference CLI's decode route (cli.cpp:277-376) on the B200:
    gen -> decode with the UNMODIFIED reference decoders (cpu:) and with the
    CUDA decoder -> compare the hypothesis JSONL files: WER 0, exit code 0."""
    if not os.path.exists(CLI):
        pytest.skip("tools/rnntg_cli not built (needs the reference headers)")
    data = str(tmp_path / "data")

    def run(*args):
        r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (args, r.stdout, r.stderr)
        return r.stdout

    run("gen", "--out", data, "--batch", "6", "--frames", "20", "--feature-dim", "12", "--vocab", "14",
        "--max-symbols", "4", "--seed", "11")
    common = ["--data", data, "--model", model, "--hidden-dim", "32", "--joint-dim", "24", *extra]
    run("decode", *common, "--algo", "cpu:" + algo, "--hyp", str(tmp_path / "ref.jsonl"))
    out = run("decode", *common, "--algo", algo, "--exec", exec_, "--hyp", str(tmp_path / "gpu.jsonl"),
              "--iters", "2")
    assert '"joint_evals"' in out
    cmp = subprocess.run([CLI, "compare", str(tmp_path / "ref.jsonl"), str(tmp_path / "gpu.jsonl")],
                         capture_output=True, text=True)
    assert cmp.returncode == 0 and cmp.stdout.strip() == "WER 0", cmp.stdout + cmp.stderr
