"""TEST INFRASTRUCTURE: decimal matrix I/O golden cases
(tests/golden/io_reference.json): the reference's own matrix_to_json /
matrix_to_csv text (precision.py:252-341) for matrices it produced, with
their exact word expansions.  Runs the UNMODIFIED reference under
oracle/gmpy2_shim; only in the build container (needs /root/reference).

    python oracle/make_golden_io.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (shim + reference on sys.path)
from mpps import coefficients, engine, gallery, precision  # noqa: E402


def cwords(A):
    return [[[mg.words(e.real), mg.words(e.imag)] for e in row] for row in A.rows]


def case(name, A):
    return {"name": name, "digits": A.produced_at.decimal_digits, "words": cwords(A),
            "json": precision.matrix_to_json(A), "csv": precision.matrix_to_csv(A)}


def main():
    ctx31, ctx15, ctx63, ctx7 = (precision.PrecisionCtx(d) for d in (31, 15, 63, 7))
    out = []
    out.append(case("smoke4_d31", precision.round_to(gallery.gen_smoke(4, ctx31), ctx31)))
    out.append(case("exp30_d31", engine.ps_mixed_exp(precision.MPMatrix(mg.synth(4, 1.0, 0).tolist(), ctx31), 30,
                                                     ctx31).result))
    out.append(case("exp16_d15", engine.ps_mixed_exp(precision.MPMatrix(mg.synth(4, 0.5, 1).tolist(), ctx15), 16,
                                                     ctx15).result))
    num, _ = coefficients.pade_exp_coeffs(26, 26)
    out.append(case("pade26_d63", engine.ps_mixed_general(precision.MPMatrix(mg.synth(3, 2.0, 2).tolist(), ctx63),
                                                          num, ctx63).result))
    out.append(case("round_d7", precision.round_to(precision.MPMatrix(mg.synth(3, 3.0, 4).tolist(), ctx15), ctx7)))
    neg = precision.MPMatrix([[complex(-1.5e-300, 2.0), 0.0], [complex(0.0, -3.25e10), 7.0]], ctx31)
    out.append(case("signs_d31", neg))
    path = os.path.join(mg.OUT, "io_reference.json")
    with open(path, "w") as f:
        json.dump({"source": "mpps.precision.matrix_to_json / matrix_to_csv (reference, under the gmpy2 shim)",
                   "cases": out}, f)
    print("wrote", path)


if __name__ == "__main__":
    main()
