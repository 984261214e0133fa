"""Gallery generators and the command-line front end (gallery.py, cli.py).

Golden data: tests/golden/cli_reference.json, written by the unmodified
reference under the gmpy2 shim (oracle/make_golden_cli.py): the exact
entries of every generator and the stdout of ``mpps plan|table1|eval``.

CPU tests: generator entries bit-exact, argument errors and exit codes.
GPU tests: the same command lines through ``paper_2312_17396_b200.cli.main``
-- schedules, counters and cost ratios exactly equal, result entries within
10 r n 10^-d of the reference's, the CSV/JSON document layout identical --
and the device acceptance restatement (``verify``) passing."""
import contextlib
import io
import json
import os
from fractions import Fraction

import pytest

from paper_2312_17396_b200 import cli, gallery
from paper_2312_17396_b200.precision import PrecisionCtx

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli_reference.json")))


def _fr(ws):
    return sum((Fraction(w) for w in ws), Fraction(0))


def run(argv):
    buf, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return code, buf.getvalue(), err.getvalue()


@pytest.mark.parametrize("case", GOLD["gallery"], ids=lambda c: f"{c['name']}{c['n']}_d{c['digits']}")
def test_gallery_entries_bit_exact(case):
    ctx = PrecisionCtx(case["digits"])
    got = gallery.generate_values(case["name"], case["n"], case["seed"], case["scale"], ctx)
    want = [[(_fr(e[0]), _fr(e[1])) for e in row] for row in case["words"]]
    assert got == want


def test_gallery_errors():
    with pytest.raises(ValueError):
        gallery.gen_cauchy(0)
    with pytest.raises(KeyError):
        gallery.generate_values("nope", 3)


def test_scale_and_round_values_exact():
    v = gallery.gen_cauchy(3, PrecisionCtx(31))
    s = gallery.scale_values(v, 3)
    assert all(a[0] == b[0] / 8 for ra, rb in zip(s, v) for a, b in zip(ra, rb))
    r = gallery.round_values(v, PrecisionCtx(7))
    assert r[0][1][0] == Fraction(11184811, 33554432)       # RN_24(1/3)
    assert r[0][2][0] == Fraction(1, 4) and r[0][0][0] == Fraction(1, 2)


def test_cli_usage_errors():
    code, _, err = run(["eval", "--matrix", "no_such_generator", "--digits", "15"])
    assert code == cli.EXIT_USAGE and "unknown matrix" in err
    code, _, err = run(["table1", "--matrix", "cauchy", "--digits-list", "15,x"])
    assert code == cli.EXIT_USAGE and "malformed" in err
    code, _, err = run(["table1", "--matrix", __file__, "--digits-list", "15"])
    assert code == cli.EXIT_USAGE and "named generator" in err
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["eval"])        # --matrix is required


def test_table_to_csv_layout():
    rows = [{"digits": 32, "m": 42, "s": 7, "r": 6, "schedule": [29, 23, 16, 7, 1, 1], "cost_ratio": 0.70047,
             "savings": 0.29953}]
    assert cli.table_to_csv(rows).splitlines() == ["digits,m,s,r,schedule,cost_ratio,savings",
                                                   "32,42,7,6,29 23 16 7 1 1,0.7005,0.2995"]


# ----------------------------------------------------------------- GPU
def _runs(cmd):
    return [r for r in GOLD["cli"] if r["argv"][0] == cmd]


def _close_str(a, b, rel=1e-5):
    fa, fb = float(a), float(b)
    return abs(fa - fb) <= rel * max(abs(fa), abs(fb), 1e-300)


def _check_plan(got, want):
    for k in ("s", "r", "nu", "working_digits", "digits", "delta", "fix_params", "degenerate_levels", "nilpotent",
              "explicit_powers"):
        assert got[k] == want[k], k
    assert got["roundoffs"] == want["roundoffs"]
    for k in ("tau", "norm_bs"):
        assert len(got[k]) == len(want[k])
        assert all(_close_str(a, b) for a, b in zip(got[k], want[k])), k
    assert _close_str(got["norm_y"], want["norm_y"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", _runs("plan"), ids=lambda c: "_".join(c["argv"][2:6]))
def test_cli_plan_matches_reference(cuda, case):
    code, out, err = run(case["argv"])
    assert code == case["exit"] == 0, err
    got, want = json.loads(out), json.loads(case["stdout"])
    _check_plan(got, want)
    assert got["cost_ratio"] == want["cost_ratio"] and got["savings"] == want["savings"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", _runs("table1"), ids=lambda c: c["argv"][-1])
def test_cli_table1_matches_reference(cuda, case):
    code, out, err = run(case["argv"])
    assert code == case["exit"] == 0, err
    if "csv" in case["argv"]:
        assert out == case["stdout"]            # schedules and 4-decimal ratios, byte for byte
    else:
        assert json.loads(out) == json.loads(case["stdout"])


def _entries(doc_matrix):
    return [Fraction(e) if "j" not in e else None for e in doc_matrix["entries"]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", _runs("eval"), ids=lambda c: "_".join(c["argv"][2:4]))
def test_cli_eval_matches_reference(cuda, case):
    code, out, err = run(case["argv"])
    assert code == case["exit"] == 0, err
    argv = case["argv"]
    d = int(argv[argv.index("--digits") + 1])
    if "csv" in argv:
        g_csv, g_rep = out.split("\n\n", 1)
        w_csv, w_rep = case["stdout"].split("\n\n", 1)
        gl, wl = g_csv.strip().splitlines(), w_csv.strip().splitlines()
        assert gl[0] == wl[0] == f"digits,{d}"
        got_vals = [Fraction(x) for line in gl[1:] for x in line.split(",")]
        want_vals = [Fraction(x) for line in wl[1:] for x in line.split(",")]
        got_rep, want_rep = json.loads(g_rep), json.loads(w_rep)
        n = len(gl) - 1
    else:
        g, w = json.loads(out), json.loads(case["stdout"])
        assert {k: g["matrix"][k] for k in ("n_rows", "n_cols", "decimal_digits")} == \
            {k: w["matrix"][k] for k in ("n_rows", "n_cols", "decimal_digits")}
        got_vals, want_vals = _entries(g["matrix"]), _entries(w["matrix"])
        got_rep, want_rep = g["report"], w["report"]
        n = w["matrix"]["n_rows"]
    assert set(got_rep) == set(want_rep)
    _check_plan(got_rep["plan"], want_rep["plan"])
    assert got_rep["matmuls_by_digits"] == want_rep["matmuls_by_digits"]
    assert got_rep["cost_ratio"] == want_rep["cost_ratio"]
    if "snapped_digits" in want_rep["diagnostics"]:
        assert got_rep["diagnostics"]["snapped_digits"] == want_rep["diagnostics"]["snapped_digits"]
    # normwise: ||got - want||_1 <= 10 r n 10^-d ||want||_1 (acceptance.py:197)
    cols = lambda v: [sum(abs(float(v[i * n + j])) for i in range(n)) for j in range(n)]  # noqa: E731
    diff = [a - b for a, b in zip(got_vals, want_vals)]
    r = want_rep["plan"]["r"]
    assert max(cols(diff)) <= 10 * r * n * 10.0 ** (-d) * max(cols(want_vals))


@pytest.mark.gpu
def test_cli_eval_beyond_quad_double_is_usage_error(cuda):
    code, _, err = run(["eval", "--matrix", "cauchy", "--n", "4", "--digits", "80"])
    assert code == cli.EXIT_USAGE and "quad-double" in err


@pytest.mark.gpu
def test_cli_compare_and_out_file(cuda, tmp_path):
    out = tmp_path / "cmp.json"
    code, _, err = run(["compare", "--matrix", "lotkin", "--n", "6", "--m", "16", "--digits", "15",
                        "--out", str(out)])
    assert code == 0, err
    rec = json.loads(out.read_text())
    assert rec["matrix_id"] == "lotkin" and rec["seed"] == 0
    assert rec["eps_mixed"] <= max(10 * rec["rnu"], 10 * rec["eps_fixed"])


@pytest.mark.gpu
def test_cli_file_input_roundtrip(cuda, tmp_path):
    src = tmp_path / "x.json"
    code, _, err = run(["eval", "--matrix", "cauchy", "--n", "5", "--m", "16", "--digits", "15",
                        "--out", str(src)])
    assert code == 0, err
    doc = json.loads(src.read_text())
    mfile = tmp_path / "m.json"
    mfile.write_text(json.dumps(doc["matrix"]))
    code, out, err = run(["plan", "--matrix", str(mfile), "--m", "16", "--digits", "15"])
    assert code == 0, err
    assert json.loads(out)["working_digits"] == 15


@pytest.mark.gpu
def test_cli_verify_passes(cuda):
    code, out, err = run(["verify"])
    assert code == 0, out + err
    assert out.count("[PASS]") == 6
