"""The `ttswe` tool on the GPU: the reference's harness contracts
(/root/reference/proj/tests/test_harness.cpp:46-200) with both device representations
(--rep tt = the device TT path, --rep dense = the device full-tensor path), run through the
C++ host code over the C ABI (include/ttsw/cuda_rep.hpp: CudaTTRep::compress/dense, Solver,
DenseSolver, tt_ghosted via the hooks)."""
import csv
import io
import json
import math
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2408_03483_b200", "ttswe")
HEADER = "case,scheme,rep,N,dt,steps,l2_c1,l2_c2,l2_c3,rel_l2_c1,order_c1,max_rank,wall_s,eps_min,eps_max"


def tool(*args, timeout=900):
    p = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def report(*args):
    rc, out, err = tool(*args)
    assert rc == 0, err
    rows = list(csv.DictReader(io.StringIO(out)))
    return rows


def test_kelvin_upwind5_smoke_contract():
    # test_harness.cpp:62-85
    d = report("run", "--case", "kelvin", "--scheme", "upwind5", "--rep", "dense", "--n", "40")[0]
    _, out, _ = tool("cases", "--case", "kelvin", "--what", "spec")
    T = float(out.split(",")[4])
    dt = 2.5e-4 * (1.0 / 40) ** (5.0 / 3.0)
    assert int(d["steps"]) == math.ceil(T / dt)
    l2 = float(d["l2_c1"])
    assert math.isfinite(l2) and l2 > 0
    t = report("run", "--case", "kelvin", "--scheme", "upwind5", "--rep", "tt", "--n", "40")[0]
    assert float(t["l2_c1"]) <= 2.0 * l2
    assert int(t["max_rank"]) <= 20
    assert float(t["eps_max"]) >= float(t["eps_min"]) > 0


def test_manufactured_dense_convergence_order():
    # test_harness.cpp:87-100: halving the grid spacing divides the error by about 2^p
    rows = report("convergence", "--case", "manufactured", "--scheme", "upwind5", "--rep", "dense",
                  "--grids", "40,80")
    assert len(rows) == 2
    order = float(rows[1]["order_c1"])
    assert 4.3 < order < 5.9, order
    assert float(rows[0]["rel_l2_c1"]) == 1.0 and float(rows[1]["rel_l2_c1"]) < 1.0


@pytest.mark.parametrize("rep", ["dense", "tt"])
def test_zero_step_run_reproduces_the_ic(rep):
    # test_harness.cpp:102-116
    r = report("run", "--case", "inertia-gravity", "--scheme", "upwind3", "--rep", rep, "--n", "24",
               "--final-time", "0")[0]
    assert int(r["steps"]) == 0
    for c in ("l2_c1", "l2_c2", "l2_c3"):
        assert float(r[c]) <= 1e-8


def test_cli_run_writes_csv(tmp_path):
    # test_harness.cpp:124-141
    out = tmp_path / "ttswe_run.csv"
    rc, _, err = tool("run", "--case", "kelvin", "--scheme", "upwind5", "--rep", "dense", "--n", "20",
                      "--out", str(out))
    assert rc == 0, err
    lines = out.read_text().splitlines()
    assert lines[0] == HEADER
    assert lines[1].startswith("kelvin,")


def test_cli_convergence_rows_and_orders(tmp_path):
    # test_harness.cpp:143-166 (TT, WENO5 via the device TT-cross)
    out = tmp_path / "ttswe_convergence.csv"
    rc, _, err = tool("convergence", "--case", "manufactured", "--scheme", "weno5", "--rep", "tt",
                      "--grids", "16,32,64", "--out", str(out))
    assert rc == 0, err
    rows = list(csv.reader(out.read_text().splitlines()))[1:]
    assert len(rows) == 3
    assert sum(1 for r in rows if r[10] != "") == 2


def test_cli_json_mirrors_csv(tmp_path):
    # test_harness.cpp:168-186
    out = tmp_path / "ttswe_json.csv"
    rc, _, err = tool("run", "--case", "inertia-gravity", "--scheme", "upwind3", "--rep", "tt", "--n", "16",
                      "--json", "--out", str(out))
    assert rc == 0, err
    doc = json.loads((tmp_path / "ttswe_json.csv.json").read_text())
    assert isinstance(doc, list) and len(doc) == 1
    for key in HEADER.split(","):
        assert key in doc[0]
    assert doc[0]["case"] == "inertia-gravity" and doc[0]["rep"] == "tt"


def test_cli_identical_configuration_and_seed_reproduce_the_report(tmp_path):
    # test_harness.cpp:188-199: determinism of the TT path (cross seed, batched roundings)
    rows = []
    for k in range(2):
        out = tmp_path / f"det{k}.csv"
        rc, _, err = tool("run", "--case", "manufactured", "--scheme", "weno5", "--rep", "tt", "--n", "16",
                          "--seed", "7", "--out", str(out))
        assert rc == 0, err
        r = out.read_text().splitlines()
        rows.append([",".join(f if i != 12 else "-" for i, f in enumerate(line.split(","))) for line in r])
    assert rows[0] == rows[1]


def test_cuda_rep_names_and_kelvin_tt_tracks_dense():
    # --rep cuda / cuda-dense name the same device paths; the Dirichlet (Kelvin) TT run stays
    # close to the dense one (both against the exact solution)
    t = report("run", "--case", "kelvin", "--scheme", "upwind3", "--rep", "cuda", "--n", "32")[0]
    d = report("run", "--case", "kelvin", "--scheme", "upwind3", "--rep", "cuda-dense", "--n", "32")[0]
    assert t["rep"] == "cuda" and d["rep"] == "cuda-dense"
    assert t["steps"] == d["steps"]
    assert float(t["l2_c1"]) <= 2.0 * float(d["l2_c1"])
