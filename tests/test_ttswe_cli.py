"""CPU checks of the `ttswe` host tool (paper_2408_03483_b200/host): the case table and exact /
manufactured cell averages against a numpy restatement of proj/src/cases.cpp:11-266, and the
CLI's configuration errors (exit 1) and help (exit 0) of proj/tests/test_harness.cpp:172-178 —
none of these touch the GPU."""
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2408_03483_b200", "ttswe")


def tool(*args):
    p = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout, p.stderr


def values(*args):
    rc, out, err = tool(*args)
    assert rc == 0, err
    return np.array([float(v) for v in out.strip().split(",")])


def gauss(nq):
    if nq == 2:
        a = 1 / (2 * math.sqrt(3))
        return [-a, a], [0.5, 0.5]
    b = math.sqrt(3 / 5) / 2
    return [-b, 0.0, b], [5 / 18, 8 / 18, 5 / 18]


def averages(fn, n, nq, lo=0, hi=None):
    hi = n if hi is None else hi
    off, w = gauss(nq)
    dx = 1.0 / n
    out = np.zeros((hi - lo, hi - lo))
    for a in range(nq):
        for b in range(nq):
            xc = (np.arange(lo, hi) + 0.5) * dx + off[a] * dx
            yc = (np.arange(lo, hi) + 0.5) * dx + off[b] * dx
            X, Y = np.meshgrid(xc, yc, indexing="ij")
            out += w[a] * w[b] * fn(X, Y)
    return out


def spec(name):
    _, out, _ = tool("cases", "--case", name, "--what", "spec")
    f = out.strip().split(",")
    return dict(g=float(f[1]), f=float(f[2]), H=float(f[3]), T=float(f[4]), L=float(f[5]))


def test_case_table_nondimensional_parameters():
    # Nondimensionalizer (cases.hpp:28-57): g U^-2 H*, f L/U, H / H*; final time T U / L
    k = spec("kelvin")
    assert k["g"] == pytest.approx(10 / (5e-3 ** 2 / 0.1), rel=1e-15) and k["f"] == pytest.approx(1e-4 / (5e-3 / 5e6))
    assert k["H"] == pytest.approx(1000 / 0.1) and k["T"] == pytest.approx(3 * 3600 / (5e6 / 5e-3)) and k["L"] == 1
    m = spec("manufactured")
    assert m["H"] == pytest.approx(2.0) and m["T"] == pytest.approx(3 * 3600 / 1e9)
    for name in ("inertia-gravity", "barotropic-tide"):
        assert spec(name)["L"] == 1


def test_kelvin_exact_averages_match_numpy():
    s = spec("kelvin")
    c = math.sqrt(s["g"] * s["H"])
    rossby = c / s["f"]
    t = 0.3 * s["T"]

    def eta(x, y):
        wave = 1e-4 * np.sin(2 * math.pi * (y + c * t)) + 2e-4 * np.sin(4 * math.pi * (y + c * t))
        return -s["H"] * wave * np.exp(-x / rossby)

    want = averages(eta, 20, 3)
    got = values("cases", "--case", "kelvin", "--n", "20", "--t", repr(t), "--component", "0").reshape(20, 20, order="F")
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def test_manufactured_source_averages_match_numpy():
    s = spec("manufactured")
    A = 1e-2 / 500.0
    B = 1e-2 / 1e-2
    kx = ky = 2 * math.pi
    c = math.sqrt(s["g"] * s["H"])
    om = math.sqrt(c * c * (kx * kx + ky * ky))
    t = 0.5 * s["T"]

    def src(comp):
        def f(x, y):
            ph = kx * x + ky * y - om * t
            cp, sp = np.cos(ph), np.sin(ph)
            h = s["H"] + A * sp
            if comp == 0:
                return -om * A * cp + kx * B * (A * cp * cp - h * sp)
            if comp == 1:
                return (B * om * (-A * cp * cp + h * sp) + kx * B * B * (A * cp ** 3 - 2 * h * cp * sp)
                        + s["g"] * h * A * kx * cp)
            return s["g"] * h * A * ky * cp + s["f"] * h * B * cp
        return f

    n = 16
    got = values("cases", "--case", "manufactured", "--n", str(n), "--t", repr(t), "--what", "source")
    for comp in range(3):
        want = averages(src(comp), n, 3)
        g = got[comp * n * n:(comp + 1) * n * n].reshape(n, n, order="F")
        assert np.abs(g - want).max() <= 1e-12 * np.abs(want).max(), comp


def test_tide_strips_are_exact_ghost_cell_averages():
    # exact_strips = exact cell averages of the ghost rows / columns (tt_ghosted strips,
    # cases.cpp:310-343), barotropic tide v component (cases.cpp:178-186)
    s = spec("barotropic-tide")
    n, t = 16, 0.4 * s["T"]
    modes = [(0.2 / 0.2, 2.5 * math.pi), (0.4 / 0.2, 4.5 * math.pi)]

    def v(x, y):
        out = 0.0 * x
        for amp, kx in modes:
            om = math.sqrt(s["g"] * s["H"] * kx * kx + s["f"] ** 2)
            a = s["g"] * amp * kx / (om * om - s["f"] ** 2)
            out = out + a * s["f"] * np.sin(kx * x) * np.cos(om * t)
        return out

    full = averages(v, n, 3, lo=-3, hi=n + 3)
    rows = [0, 1, 2, n + 3, n + 4, n + 5]
    st = values("cases", "--case", "barotropic-tide", "--n", str(n), "--t", repr(t), "--component", "2",
                "--what", "strips")
    sx = st[:6 * (n + 6)].reshape(6, n + 6, order="F")
    sy = st[6 * (n + 6):].reshape(n + 6, 6, order="F")
    scale = np.abs(full).max()
    assert np.abs(sx - full[rows, :]).max() <= 1e-13 * scale
    assert np.abs(sy - full[:, rows]).max() <= 1e-13 * scale


@pytest.mark.parametrize("args", [["convergence", "--case", "kelvin", "--grids", "40,100"],
                                  ["run", "--case", "unknown-case"],
                                  ["run", "--definitely-not-a-flag", "3"],
                                  ["run", "--case", "kelvin", "--n", "8"],
                                  ["convergence", "--case", "kelvin", "--grids", "40"],
                                  ["run", "--rep", "sparse"],
                                  ["nonsense"]])
def test_configuration_errors_exit_1(args):
    rc, _, _ = tool(*args)
    assert rc == 1, args


def test_help_exits_0():
    rc, out, _ = tool("--help")
    assert rc == 0 and "run" in out and "convergence" in out
