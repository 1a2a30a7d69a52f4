"""The command-line drivers (paper_1808_04580_b200/cli, tools/commands.cpp
analogue: eigs, cluster, bench): exit codes, the fgs-report-v1 report
(validated against the reference's own schema/report.schema.json where the
reference tree is present) and CSV handling.  CPU only: nothing here touches
the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
EXE = os.path.join(os.path.dirname(HERE), "paper_1808_04580_b200", "fgs-b200")


@pytest.fixture(scope="module")
def exe():
    from paper_1808_04580_b200 import build
    build.build()
    assert os.path.exists(EXE)
    return EXE


def run(exe, *args):
    return subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=120)


def write_spiral_csv(path, per_class=400, classes=5, seed=4):
    """a labelled 3-D spiral cloud in the reference's CSV layout
    (x0,x1,x2,label; dataset.cpp save_points_csv) for the CLI tests"""
    rng = np.random.default_rng(seed)
    rows = []
    for c in range(classes):
        t = rng.uniform(0.0, 1.0, per_class)
        ang = 4.0 * np.pi * t + 2.0 * np.pi * c / classes
        pts = np.stack([(2.0 + 8.0 * t) * np.cos(ang), (2.0 + 8.0 * t) * np.sin(ang), 10.0 * t], axis=1)
        pts += 0.3 * rng.standard_normal(pts.shape)
        rows.append(np.column_stack([pts, np.full(per_class, c)]))
    data = np.vstack(rows)
    with open(path, "w") as f:
        f.write("x0,x1,x2,label\n")
        for r in data:
            f.write(f"{float(r[0])!r},{float(r[1])!r},{float(r[2])!r},{int(r[3])}\n")


def check_report(rep):
    """schema/report.schema.json constraints, restated (the -m gpu tests run
    where the reference tree is absent; test_report_matches_reference_schema
    checks the restatement against the file itself)."""
    for key in ("schema", "command", "parameters", "seed", "metrics", "timings_seconds", "status"):
        assert key in rep, key
    assert rep["schema"] == "fgs-report-v1"
    assert isinstance(rep["command"], str) and isinstance(rep["parameters"], dict)
    assert isinstance(rep["seed"], int) and rep["seed"] >= 0
    assert all(isinstance(v, (int, float)) for v in rep.get("eigenvalues", []))
    for name, m in rep["metrics"].items():
        assert set(m) >= {"value", "definition"} and isinstance(m["definition"], str), name
        assert isinstance(m["value"], (int, float, list))
    assert all(isinstance(v, (int, float)) and v >= 0 for v in rep["timings_seconds"].values())
    assert rep["status"] in ("ok", "numerical-failure")
    assert isinstance(rep.get("diagnostic", ""), str)
    if "extra" in rep:
        assert isinstance(rep["extra"], dict)


def test_usage_errors_exit_2(exe, tmp_path):
    assert run(exe).returncode == 2
    # commands outside the hot path's scope are usage errors
    for cmd in ("gen", "segment", "ssl-kernel", "krr", "ssl-pf"):
        assert run(exe, cmd, "--out", tmp_path / "x.csv").returncode == 2
    assert run(exe, "eigs", "--out", tmp_path / "r.json").returncode == 2  # --in required
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--bogus", 1).returncode == 2
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--setup", 4).returncode == 2
    assert run(exe, "eigs", "--in", "a.csv", "--out", "r.json", "--kernel", "cosine").returncode == 2
    assert run(exe, "bench", "--out", "r.json", "--methods", "magic").returncode == 2
    assert run(exe, "--help").returncode == 0


def test_csv_input_errors_exit_2(exe, tmp_path):
    cases = {"empty.csv": "", "noheader.csv": "\n1,2\n", "ragged.csv": "x0,x1\n1,2\n3\n",
             "nonnum.csv": "x0,x1\n1,abc\n", "inf.csv": "x0,x1\n1,inf\n", "norows.csv": "x0,x1\n",
             "badlabel.csv": "x0,label\n1,2.5\n"}
    for name, text in cases.items():
        p = tmp_path / name
        p.write_text(text)
        r = run(exe, "eigs", "--in", p, "--out", tmp_path / "r.json")
        assert r.returncode == 2 and "input error" in r.stderr, (name, r.stderr)
    r = run(exe, "eigs", "--in", tmp_path / "missing.csv", "--out", tmp_path / "r.json")
    assert r.returncode == 2 and "cannot open" in r.stderr


REF_SCHEMA = "/root/reference/proj/schema/report.schema.json"


def _validate(inst, schema, path="$"):
    """the draft-07 subset the reference schema uses: type, enum, required,
    properties, additionalProperties, items, minimum"""
    types = schema.get("type")
    if types is not None:
        ok = {"object": dict, "array": list, "string": str, "integer": int, "number": (int, float)}
        tl = types if isinstance(types, list) else [types]
        assert any(isinstance(inst, ok[t]) and not (t in ("integer", "number") and isinstance(inst, bool))
                   for t in tl), (path, types, inst)
    if "enum" in schema:
        assert inst in schema["enum"], (path, inst)
    if "minimum" in schema:
        assert inst >= schema["minimum"], (path, inst)
    if isinstance(inst, dict):
        for k in schema.get("required", []):
            assert k in inst, (path, k)
        props = schema.get("properties", {})
        for k, v in inst.items():
            if k in props:
                _validate(v, props[k], f"{path}.{k}")
            elif isinstance(schema.get("additionalProperties"), dict):
                _validate(v, schema["additionalProperties"], f"{path}.{k}")
    if isinstance(inst, list) and "items" in schema:
        for i, v in enumerate(inst):
            _validate(v, schema["items"], f"{path}[{i}]")


@pytest.mark.skipif(not os.path.exists(REF_SCHEMA), reason="reference tree not present")
def test_report_matches_reference_schema(exe, tmp_path):
    # the CLI's report, a numerical-failure report and a usage of every
    # metric shape, validated against proj/schema/report.schema.json itself
    schema = json.load(open(REF_SCHEMA))
    p = tmp_path / "far.csv"
    p.write_text("x0\n0\n1000\n1000.5\n")
    rep_path = tmp_path / "fail.json"
    r = run(exe, "eigs", "--in", p, "--out", rep_path, "--sigma", 0.01, "--k", 1, "--method", "direct")
    assert r.returncode in (1, 2)
    if rep_path.exists():
        rep = json.loads(rep_path.read_text())
        _validate(rep, schema)
        check_report(rep)
    # the restated checker accepts exactly what the schema accepts on
    # hand-made reports (one valid, several invalid)
    good = {"schema": "fgs-report-v1", "command": "eigs", "parameters": {}, "seed": 3,
            "metrics": {"a": {"value": 1.5, "definition": "x"}, "b": {"value": [1, 2], "definition": "y"}},
            "timings_seconds": {"setup": 0.1}, "status": "ok", "eigenvalues": [1.0, 0.5]}
    _validate(good, schema)
    check_report(good)
    for bad in ({**good, "schema": "v2"}, {**good, "seed": -1}, {**good, "status": "fine"},
                {**good, "timings_seconds": {"setup": -1.0}},
                {**good, "metrics": {"a": {"value": 1.0}}}):
        with pytest.raises(AssertionError):
            _validate(bad, schema)
        with pytest.raises(AssertionError):
            check_report(bad)

