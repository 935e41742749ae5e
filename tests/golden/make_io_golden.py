"""Golden fixtures for the reference's text formats:
runs the UNMODIFIED reference (oracle/_ref/libcmtf_ref.so) on a set of COO
text files -- valid ones and every ParseError / ValidationError path of
parse_coo_file / load_tensor / load_matrix (src/sparse_data.cpp:66-277) --
plus save_tensor and save_model (src/model_io.cpp:94-126), and records what
the reference returns or throws.  tests/test_io.py holds the product's
parser / writers (paper_1708_08640_b200/io.py -> csrc/io.cpp) to these.

    python tests/golden/make_io_golden.py
"""
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

# (name, text, kind, extra): kind "tensor" or "matrix" (extra: mode, weight, dims)
TENSOR_CASES = [
    ("header_comments_crlf", "# a comment\n3 4 5\n1 1 1 0.5\r\n\n2 3 4 -1.25e3 # trailing\n"
                             "\t3 4 5\t7\n", {}),
    ("no_header_inferred", "1 1 1 0.5\n2 3 4 -1.25e3\n7 2 9 1e-3\n", {}),
    ("header_only", "5 6 7\n", {}),
    ("single_all_int_line", "1 2 3 4\n", {}),
    ("single_entry", "1 2 3 4.5\n", {}),
    ("header_two_dims", "3 3\n1 2 0.25\n3 3 -2\n", {}),
    ("order4", "2 2 2 2\n1 1 1 1 1\n2 2 2 2 2\n1 2 1 2 3.5\n", {}),
    ("field_count", "1 1 1 0.5\n2 3 0.5\n", {}),
    ("field_count_more", "3 3 3\n1 1 1 1\n1 2 3 4 5\n", {}),
    ("bad_index_alpha", "1 1 1 0.5\n1 a 1 2\n", {}),
    ("bad_index_plus", "1 1 1 0.5\n1 +2 1 2\n", {}),
    ("bad_index_neg", "1 1 1 0.5\n1 -2 1 2\n", {}),
    ("bad_index_zero", "1 1 0 2\n", {}),
    ("bad_index_big", "1 1 4294967296 2\n", {}),
    ("index_max", "1 1 4294967295 2\n", {}),
    ("bad_index_float", "1 1 1.0 2\n", {}),
    ("bad_value_alpha", "1 1 1 x\n", {}),
    ("bad_value_underflow", "1 1 1 1e-400\n", {}),
    ("bad_value_overflow", "1 1 1 1e400\n", {}),
    ("bad_value_subnormal", "1 1 1 1e-310\n", {}),
    ("bad_value_inf", "1 1 1 inf\n", {}),
    ("bad_value_nan", "1 1 1 nan\n", {}),
    ("value_hex", "1 1 1 0x1p3\n2 2 2 1.5e+2\n", {}),
    ("value_forms", "1 1 1 .5\n2 2 2 -0\n3 3 3 +7\n4 4 4 1E2\n", {}),
    ("value_trailing", "1 1 1 2.5x\n", {}),
    ("one_token_entry", "7\n", {}),
    ("one_token_then_more", "7\n1 2\n", {}),
    ("order1", "1 2.0\n2 3.0\n", {}),
    ("empty", "", {}),
    ("only_comments", "# nothing\n\n   \n", {}),
    ("header_bad", "0 5 5\n1 1 1 2\n", {}),
    ("header_plus", "+5 5 5\n1 1 1 2\n", {}),
    ("duplicate", "3 3 3\n1 2 3 0.5\n2 2 2 1\n1 2 3 0.7\n", {}),
    ("duplicate_two", "3 3 3\n3 3 3 1\n1 2 3 0.5\n3 3 3 0.1\n1 2 3 0.7\n", {}),
    ("out_of_range", "3 3 3\n1 2 3 0.5\n4 1 1 1\n", {}),
    ("crlf_header", "2 2 2\r\n1 1 1 1\r\n2 2 2 2\r\n", {}),
]
MODEL_ERROR_CASES = [
    "", "CORE\n", "CORE\n2 2\n1 2 3\n", "CORE\n1 1\n1 x\n", "CORE\n0 1\n", "CORE\n-1 1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1\n1\nBOGUS\n",
    "CORE\n1 1\n1\nFOO 1\n1 1\n1\n", "CORE\n1 1\n1\nFACTOR 2\n1 1\n1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1 1\n", "CORE\n1 1\n1 2\nFACTOR 1\n1 1\n1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1\n1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 2\n1 1\nFACTOR 2\n1 1\n1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1\n1\nFACTOR 2\n1 1\n1\nCOUPLED 3\n1 1\n1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1\n1\nFACTOR 2\n1 1\n1\nCOUPLED 1\n2 2\n1 1 1 1\n",
    "CORE\n1 1\n1\nFACTOR 1\n1 1\n1\nFACTOR 2\n1 1\n1\nCOUPLED 2\n2 1\n1 1\n",
    "CORE\n1 1\n0x1p-2\nFACTOR 1\n1 1\n5abc\n",
    "CORE\r\n1  1\r\n 1\r\nFACTOR 1\n1 1\n1\nFACTOR 2\n1 1\n 1 \n\n",
]
MATRIX_CASES = [
    ("matrix_ok_header", "4 3\n1 1 0.5\n4 3 -1\n", {"mode": 1, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_ok_noheader", "1 1 0.5\n2 7 -1\n", {"mode": 2, "weight": 2.0, "dims": [4, 5, 6]}),
    ("matrix_header_rows", "3 3\n1 1 0.5\n", {"mode": 1, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_row_exceeds", "1 1 0.5\n9 1 1\n", {"mode": 1, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_mode_range", "1 1 0.5\n", {"mode": 4, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_mode_zero", "1 1 0.5\n", {"mode": 0, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_weight", "1 1 0.5\n", {"mode": 1, "weight": 0.0, "dims": [4, 5, 6]}),
    ("matrix_order3", "1 1 1 0.5\n", {"mode": 1, "weight": 10.0, "dims": [4, 5, 6]}),
    ("matrix_duplicate", "4 3\n1 1 0.5\n2 2 1\n1 1 0.7\n", {"mode": 1, "weight": 10.0,
                                                           "dims": [4, 5, 6]}),
    ("matrix_header_only", "4 3\n", {"mode": 1, "weight": 10.0, "dims": [4, 5, 6]}),
]


def big_text(seed=7, n=120_000, bad_line=None):
    """A multi-megabyte file (the product parses it in parallel chunks):
    header, comments every 1000 lines, mixed value formats."""
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = [5000, 4000, 300]
    seen = set()
    lines = ["# big file", " ".join(map(str, dims))]
    while len(seen) < n:
        t = (int(rng.integers(1, dims[0] + 1)), int(rng.integers(1, dims[1] + 1)),
             int(rng.integers(1, dims[2] + 1)))
        if t in seen:
            continue
        seen.add(t)
        v = float(rng.normal() * 10.0 ** int(rng.integers(-5, 6)))
        k = len(seen)
        s = repr(v) if k % 3 else ("%.6e" % v if k % 2 else "%.17g" % v)
        lines.append(f"{t[0]} {t[1]} {t[2]} {s}")
        if k % 1000 == 0:
            lines.append("# block %d" % k)
    if bad_line is not None:
        lines[bad_line - 1] = "1 2 zz 3"
    return "\n".join(lines) + "\n"


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(res, path):
    if res[0] != "ok":
        return {"error": res[0], "message": res[1].replace(path, "{path}")}
    _, dims, idx, vals = res
    return {"dims": dims, "idx": idx.reshape(-1).tolist(), "vals": [v.hex() for v in vals]}


def main():
    O.build()
    tmp = tempfile.mkdtemp()
    out = {"tensor": [], "matrix": [], "big": [], "save": {}}
    for name, text, _ in TENSOR_CASES:
        path = os.path.join(tmp, name + ".tns")
        open(path, "w", newline="").write(text)
        out["tensor"].append({"name": name, "text": text, **outcome(O.ref_load(path), path)})
    for name, text, ex in MATRIX_CASES:
        path = os.path.join(tmp, name + ".mat")
        open(path, "w", newline="").write(text)
        res = O.ref_load(path, True, ex["mode"], ex["weight"], ex["dims"])
        out["matrix"].append({"name": name, "text": text, "mode": ex["mode"],
                              "weight": ex["weight"], "tensor_dims": ex["dims"],
                              **outcome(res, path)})
    for seed, bad in [(7, None), (8, 77_777), (9, 3)]:
        path = os.path.join(tmp, f"big{seed}.tns")
        open(path, "w").write(big_text(seed, bad_line=bad))
        res = O.ref_load(path)
        rec = {"seed": seed, "bad_line": bad}
        if res[0] == "ok":
            rec.update({"dims": res[1], "nnz": int(res[3].shape[0]), "idx_sha": digest(res[2]),
                        "vals_sha": digest(res[3])})
        else:
            rec.update({"error": res[0], "message": res[1].replace(path, "{path}")})
        out["big"].append(rec)
    out["model_errors"] = []
    for k, text in enumerate(MODEL_ERROR_CASES):
        path = os.path.join(tmp, f"model{k}.txt")
        open(path, "w", newline="").write(text)
        r = O.ref_load_model(path)
        rec = {"text": text}
        if r[0] == "ok":
            rec.update({"order": r[1], "n_factors": r[2], "n_coupled": r[3]})
        else:
            rec.update({"error": r[0], "message": r[1].replace(path, "{path}")})
        out["model_errors"].append(rec)
    # writers: save_tensor and save_model text, byte for byte
    rng = np.random.Generator(np.random.PCG64(11))
    idx = np.array([[0, 1, 2], [3, 0, 1], [2, 2, 0]], dtype=np.uint32)
    vals = np.array([0.1, -1e-300, 12345.678901234567])
    p = os.path.join(tmp, "t.tns")
    O.ref_save_tensor(p, [4, 3, 3], idx, vals)
    out["save"]["tensor"] = {"dims": [4, 3, 3], "idx": idx.reshape(-1).tolist(),
                             "vals": [v.hex() for v in vals], "text": open(p).read()}
    core = rng.normal(size=(2, 3, 2))
    facs = [rng.normal(size=(4, 2)), rng.normal(size=(3, 3)), rng.normal(size=(5, 2))]
    cpl = [rng.normal(size=(6, 2))]
    p = os.path.join(tmp, "m.txt")
    O.ref_save_model(p, core, facs, cpl, [0])
    out["save"]["model"] = {"core": [v.hex() for v in core.reshape(-1)], "ranks": [2, 3, 2],
                            "factors": [[v.hex() for v in f.reshape(-1)] for f in facs],
                            "rows": [4, 3, 5], "couplings": [[v.hex() for v in cpl[0].reshape(-1)]],
                            "coupling_rows": [6], "coupling_modes": [0], "text": open(p).read()}
    cpcore = rng.normal(size=3)
    cfacs = [rng.normal(size=(4, 3)) for _ in range(3)]
    O.ref_save_model(p, cpcore, cfacs, cp=True)
    out["save"]["model_cp"] = {"core": [v.hex() for v in cpcore], "ranks": [3, 3, 3],
                               "factors": [[v.hex() for v in f.reshape(-1)] for f in cfacs],
                               "rows": [4, 4, 4], "text": open(p).read()}
    with open(os.path.join(HERE, "io_cases.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote io_cases.json:", len(out["tensor"]), "tensor,", len(out["matrix"]),
          "matrix cases")


if __name__ == "__main__":
    main()
