"""CLI verbs that execute on the device (reference cli.py run / ablate /
scaling), on a generated toy model: output parity with the oracle and the
ablation ladder's table."""

import numpy as np
import pytest

import oracle
from paper_1809_02697_b200 import cli, gen_model, load_model

pytestmark = pytest.mark.gpu


def test_cli_run_matches_oracle(cuda, tmp_path, capsys):
    js, wt, out = str(tmp_path / "m.json"), str(tmp_path / "m.npwt"), str(tmp_path / "o.bin")
    assert cli.main(["gen", "--kind", "resnet-block", "--depth", "2", "--channels", "16",
                     "--hw", "16", "--out", js, "--weights", wt]) == 0
    x = np.random.default_rng(3).standard_normal((1, 16, 16, 16)).astype(np.float32)
    x.tofile(tmp_path / "in.bin")
    assert cli.main(["run", "--model", js, "--weights", wt, "--mode", "fp32", "--samples", "3",
                     "--input", str(tmp_path / "in.bin"), "--out", out]) == 0
    got = np.fromfile(out, dtype="<f4").reshape(1, 16, 16, 16)
    ref = oracle.execute_reference(load_model(js, wt), {"data": x})[0]
    assert oracle.rel_err(got, ref) < 1e-4


def test_cli_ablate_and_scaling(cuda, tmp_path, capsys):
    js, wt = str(tmp_path / "m.json"), str(tmp_path / "m.npwt")
    assert cli.main(["gen", "--kind", "chain", "--depth", "3", "--channels", "32", "--hw", "28",
                     "--out", js, "--weights", wt]) == 0
    capsys.readouterr()
    assert cli.main(["ablate", "--model", js, "--weights", wt, "--mode", "bf16",
                     "--samples", "3"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert [ln.split()[0] for ln in lines[1:]] == ["baseline-nchw", "layout-opt", "transform-elim"]
    assert cli.main(["scaling", "--model", js, "--weights", wt, "--samples", "2"]) == 0
    assert capsys.readouterr().out.strip().splitlines()[0] == "gpus,samples,mean_ns,stderr_ns"
