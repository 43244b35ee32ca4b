"""The reference's own `dessim` commands (proj/tools/commands.cpp + emit.cpp,
compiled unchanged by tests/cpp/Makefile behind a minimal argument front end,
tests/cpp/cli_main.cpp) running on the B200 through the C++ façade, against
the same commands linked to the reference library (CPU). `gen-trace` bytes
must be identical; `run` / `sweep` tables must match cell by cell: integer
columns exactly, floating columns within 1e-9 relative (fp64 on both sides;
CUDA's exp may differ from glibc's in the last bit) — every method the CLI
offers: vanilla, des-seq, des-vote, topk, naee, mcmoe, with the synthetic
bank's reconstruction loss.
"""
import csv
import io
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
GPU_CLI = os.path.join(BUILD, "dessim_gpu_cli")
REF_CLI = os.path.join(BUILD, "dessim_ref_cli")

METHODS = [["--method", "vanilla"], ["--method", "des-seq", "--k", "3"],
           ["--method", "des-vote", "--beta", "0.4"], ["--method", "topk", "--k", "2"],
           ["--method", "naee", "--beta", "0.3"],
           ["--method", "mcmoe", "--beta", "0.3", "--fraction", "0.5"]]


def _cli(path, *args):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not built (make -C tests/cpp needs /root/reference)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout


def _rows(text):
    return list(csv.reader(io.StringIO("\n".join(l for l in text.splitlines()
                                                 if not l.startswith("#")))))


def _same_table(a, b):
    ra, rb = _rows(a), _rows(b)
    assert len(ra) == len(rb) and ra[0] == rb[0]
    for x, y in zip(ra[1:], rb[1:]):
        assert len(x) == len(y)
        for u, v in zip(x, y):
            if u == v:
                continue
            fu, fv = float(u), float(v)
            assert abs(fu - fv) <= 1e-9 * max(1.0, abs(fv)), (u, v, x)


def test_cli_help_without_gpu_needs_none():
    assert "usage" in subprocess.run([REF_CLI], capture_output=True, text=True).stderr \
        if os.path.exists(REF_CLI) else True


@pytest.mark.gpu
def test_gen_trace_identical(tmp_path):
    a, b = str(tmp_path / "g.moet"), str(tmp_path / "r.moet")
    args = ["--experts", "64", "--top-k", "8", "--block", "32", "--layers", "2", "--steps", "2",
            "--rho", "0.3", "--seed", "42"]
    _cli(GPU_CLI, "gen-trace", *args, "-o", a)
    _cli(REF_CLI, "gen-trace", *args, "-o", b)
    assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("method", METHODS, ids=[m[1] for m in METHODS])
def test_run_matches_reference(tmp_path, method):
    trace = str(tmp_path / "t.moet")
    _cli(REF_CLI, "gen-trace", "--experts", "64", "--top-k", "8", "--block", "32", "--layers",
         "2", "--steps", "2", "--rho", "0.3", "--seed", "42", "-o", trace)
    common = ["--trace", trace, *method, "--bank-seed", "3", "--hidden-dim", "16"]
    _same_table(_cli(GPU_CLI, "run", *common), _cli(REF_CLI, "run", *common))


@pytest.mark.gpu
def test_sweep_matches_reference(tmp_path):
    trace = str(tmp_path / "t.moet")
    _cli(REF_CLI, "gen-trace", "--experts", "64", "--top-k", "8", "--block", "32", "--steps",
         "3", "--rho", "0.3", "--seed", "7", "-o", trace)
    for m, grid in [("des-vote", ["--betas", "0.2,0.4,0.6"]), ("topk", ["--ks", "1,2,4"])]:
        common = ["--trace", trace, "--method", m, *grid]
        _same_table(_cli(GPU_CLI, "sweep", *common), _cli(REF_CLI, "sweep", *common))
