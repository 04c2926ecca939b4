"""Writes the Matrix Market parity fixtures (tests/golden/mm/*.mtx) and
records what the unmodified reference returns for each — read_matrix_market
followed by from_coo (io.hpp:50-121, tensor.hpp:118), through the oracle
shim oracle/_ref — into tests/golden/mm/expected.json. Values are stored
as float.hex (exact f64). Error messages have the file path replaced by
"{path}". Run here (where /root/reference exists):

  python tests/golden/make_mm_goldens.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

OUT = os.path.join(HERE, "mm")

B = "%%MatrixMarket matrix coordinate"
CASES = {
    # number shapes the device parses on its fast path, and ones it hands
    # to the host (long mantissa, subnormal, hex-like trailers ignored)
    "numbers_general": f"""{B} real general
% a comment line
%
4 5 12

1 1 1.
1 2 .5
1 5 -0
2 1 +2.5
2 3 1e-3\r
2 4 1E+2
3 1 0.1
3 2 0.123456789012345678901234
3 3 7 trailing tokens ignored
3 4 1.5e-310
4 5 123456789.25
4 4\t-3.75
""",
    "integer_field": f"""{B} integer general
3 3 3
1 1 7
2 2 -4
3 1 12
""",
    "pattern_symmetric": f"""{B} pattern symmetric
5 5 4
1 1
3 1
5 2
4 4
""",
    "real_symmetric": f"""{B} real symmetric
4 4 5
1 1 2.0
2 1 -1.0
3 2 -1.0
4 3 -1.0
4 4 2.0
""",
    "uppercase_header": """%%MatrixMarket MATRIX Coordinate REAL General
2 2 1
2 2 9.5
""",
    "empty_body": f"""{B} real general
6 7 0
""",
    "no_trailing_newline": f"""{B} real general
2 2 2
1 1 1.25
2 2 2.5""",
    "duplicates": f"""{B} real general
3 3 3
1 1 1.5
2 2 1.0
1 1 2.25
""",
    "err_banner": """%MatrixMarket matrix coordinate real general
1 1 0
""",
    "err_object": """%%MatrixMarket vector coordinate real general
1 1 0
""",
    "err_format": """%%MatrixMarket matrix array real general
1 1
""",
    "err_field": """%%MatrixMarket matrix coordinate complex general
1 1 0
""",
    "err_symmetry": """%%MatrixMarket matrix coordinate real hermitian
1 1 0
""",
    "err_missing_size": f"""{B} real general
% only comments
""",
    "err_bad_size": f"""{B} real general
3 three 1
""",
    "err_negative_size": f"""{B} real general
-3 3 1
""",
    "err_bad_entry": f"""{B} real general
3 3 2
1 1 1.0
1 x 2.0
""",
    "err_indented_comment": f"""{B} real general
3 3 1
 % indented comments are not comments
1 1 1.0
""",
    "err_missing_value": f"""{B} real general
3 3 2
1 1 1.0
2 2
""",
    "err_bad_value": f"""{B} real general
3 3 1
1 1 nan
""",
    "err_overflow_value": f"""{B} real general
3 3 1
1 1 1e400
""",
    "err_range_zero": f"""{B} real general
3 3 1
0 1 1.0
""",
    "err_range_high": f"""{B} real general
3 3 2
1 1 1.0
3 4 1.0
""",
    "err_count": f"""{B} real general
3 3 3
1 1 1.0
2 2 2.0
""",
    "err_empty": "",
}


def random_case(seed, m, n, k, symmetric):
    rng = np.random.default_rng(seed)
    keys = set()
    lines = []
    while len(lines) < k:
        r, c = int(rng.integers(1, m + 1)), int(rng.integers(1, n + 1))
        if symmetric and c > r:
            r, c = c, r
        if (r, c) in keys:
            continue
        keys.add((r, c))
        x = float(rng.random() * 2 - 1)
        style = len(lines) % 4
        v = f"{x:.6f}" if style == 0 else f"{x:.17g}" if style == 1 else f"{x:.3e}" if style == 2 else repr(x)
        lines.append(f"{r} {c} {v}")
    kind = "symmetric" if symmetric else "general"
    return f"{B} real {kind}\n% random\n{m} {n} {k}\n" + "\n".join(lines) + "\n"


CASES["random_general"] = random_case(1, 300, 200, 4000, False)
CASES["random_symmetric"] = random_case(2, 250, 250, 3000, True)


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = oracle.Ref()
    expected = {}
    for name, text in CASES.items():
        path = os.path.join(OUT, name + ".mtx")
        with open(path, "w", newline="") as f:
            f.write(text)
        for summ in (False, True):
            key = f"{name}:{int(summ)}"
            try:
                coo = ref.read_mm(path, sum_duplicates=summ)
                r, c, v = coo.arrays()
                expected[key] = {"shape": list(coo.shape), "row": r.tolist(), "col": c.tolist(),
                                 "val": [float(x).hex() for x in v]}
            except oracle.OracleError as e:
                msg = str(e)[len(e.kind) + 2:]
                expected[key] = {"error": e.kind, "message": msg.replace(path, "{path}")}
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(expected, f, indent=0, sort_keys=True)
    print(f"{len(expected)} cases -> {OUT}")


if __name__ == "__main__":
    main()
