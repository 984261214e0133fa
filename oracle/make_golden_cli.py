"""TEST INFRASTRUCTURE: gallery and command-line golden cases
(tests/golden/cli_reference.json).  Runs the UNMODIFIED reference under
oracle/gmpy2_shim; only in the build container (needs /root/reference).

* gallery: the exact entries of every generator (gallery.py:21-107) at the
  lattice digit counts, as exact fp64 word expansions;
* cli: stdout of ``mpps plan`` / ``mpps table1`` / ``mpps eval`` (cli.py)
  on small generated matrices, parsed as JSON.

    python oracle/make_golden_cli.py"""
import contextlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (shim + reference on sys.path)
from mpps import cli, gallery, precision  # noqa: E402


def cwords(A):
    return [[[mg.words(e.real), mg.words(e.imag)] for e in row] for row in A.rows]


GALLERY = [
    ("cauchy", 5, 0, 100.0, 15), ("cauchy", 5, 0, 100.0, 31), ("cauchy", 4, 0, 100.0, 63),
    ("cauchy", 3, 0, 100.0, 40), ("lotkin", 5, 0, 100.0, 31), ("lotkin", 4, 0, 100.0, 7),
    ("ward", 0, 0, 100.0, 15), ("nonnormal2", 0, 0, 100.0, 7), ("nonnormal2", 0, 0, 100.0, 31),
    ("triu_rand", 5, 3, 100.0, 15), ("triu_rand", 5, 4, 1.0, 31), ("triu_rand", 4, 5, 2.5, 7),
    ("smoke", 5, 0, 100.0, 63), ("smoke", 7, 0, 100.0, 15), ("smoke", 3, 0, 100.0, 7),
]

CLI = [
    ["plan", "--matrix", "cauchy", "--n", "10", "--m", "30", "--digits", "31"],
    ["plan", "--matrix", "triu_rand", "--n", "8", "--seed", "2", "--m", "16", "--digits", "15"],
    ["plan", "--matrix", "lotkin", "--n", "6", "--series", "pade_exp_num", "--m", "13", "--digits", "15",
     "--lattice", "7,15"],
    ["plan", "--matrix", "smoke", "--n", "6", "--series", "taylor_cos", "--m", "8", "--digits", "31",
     "--scale-l", "1"],
    ["table1", "--matrix", "cauchy", "--n", "20", "--m", "20", "--digits-list", "15,31,63"],
    ["table1", "--matrix", "cauchy", "--n", "20", "--digits-list", "32,64", "--m-list", "42,64",
     "--format", "csv"],
    ["table1", "--matrix", "cauchy", "--n", "100", "--digits-list", "128,256", "--m-list", "100,182"],
    ["eval", "--matrix", "cauchy", "--n", "5", "--m", "16", "--digits", "15"],
    ["eval", "--matrix", "triu_rand", "--n", "5", "--seed", "1", "--triu-scale", "1.0", "--m", "20",
     "--digits", "31", "--lattice", "7,15,31"],
    ["eval", "--matrix", "lotkin", "--n", "4", "--series", "pade_exp_den", "--m", "13", "--digits", "15"],
    ["eval", "--matrix", "ward", "--scale-l", "6", "--m", "12", "--digits", "31", "--format", "csv"],
]


def run_cli(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    return code, buf.getvalue()


def main():
    gal = []
    for name, n, seed, scale, d in GALLERY:
        ctx = precision.PrecisionCtx(d)
        A = gallery.generate(name, n, seed, scale, ctx)
        gal.append({"name": name, "n": n, "seed": seed, "scale": scale, "digits": d, "words": cwords(A)})
    runs = []
    for argv in CLI:
        code, out = run_cli(argv)
        runs.append({"argv": argv, "exit": code, "stdout": out})
    path = os.path.join(HERE, "..", "tests", "golden", "cli_reference.json")
    with open(path, "w") as f:
        json.dump({"source": "mpps.gallery generators and mpps.cli.main (unmodified reference under the "
                             "gmpy2 shim)", "gallery": gal, "cli": runs}, f)
    print("wrote", path, len(gal), "gallery cases,", len(runs), "cli runs")


if __name__ == "__main__":
    main()
