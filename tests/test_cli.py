"""CLI contract (SPEC.md [MODULE] cli, acceptance criteria 9-10): argument /
frame parsing and input errors on CPU; query / ablate / oracle records and
the JSON / CSV report schemas on the GPU."""

import csv
import io
import json
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def cli(md):
    from paper_2411_11244_b200 import cli as c

    return c


def _run(cli, capsys, *argv):
    code = cli.main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


def _write_obj(path, V, T):
    with open(path, "w") as fh:
        for v in V:
            fh.write("v " + " ".join(repr(float(x)) for x in v) + "\n")
        for t in T:
            fh.write("f " + " ".join(str(int(i) + 1) for i in t) + "\n")
    return str(path)


def test_gen_params(cli):
    assert cli.parse_gen_params("n=200,seed=3,gap=0.5,name=x,flag=true") == {
        "n": 200, "seed": 3, "gap": 0.5, "name": "x", "flag": True}
    assert cli.parse_gen_params("center=[0;0;1.5]") == {"center": (0, 0, 1.5)}
    assert cli.parse_gen_params(None) == {}
    with pytest.raises(cli.CliError):
        cli.parse_gen_params("n")


def test_frames_forms(cli, tmp_path):
    p = tmp_path / "f.json"
    p.write_text(json.dumps([{"axis": [0, 0, 1], "angle": 0.5}, None,
                             {"a": {"rotation": np.eye(3).tolist(), "translation": [1, 2, 3]}, "mesh_b": "x.obj"}]))
    fr = cli.load_frames(str(p))
    assert len(fr) == 3 and fr[1] == (None, None, None, None)
    assert fr[2][0].translation.tolist() == [1, 2, 3] and fr[2][3] == "x.obj"
    p.write_text(json.dumps({"a": [None, None], "b": [None]}))
    with pytest.raises(cli.CliError) as ei:
        cli.load_frames(str(p))
    assert "2 transforms for A but 1 for B" in str(ei.value)
    p.write_text(json.dumps([{"rotation": [[2, 0, 0], [0, 1, 0], [0, 0, 1]]}]))
    with pytest.raises(cli.CliError):
        cli.load_frames(str(p))


def test_input_errors_exit_codes(cli, capsys, tmp_path):
    bad = tmp_path / "bad.obj"
    bad.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\n")
    code, _, err = _run(cli, capsys, "query", "--mesh-a", str(bad), "--mesh-b", str(bad))
    assert code == cli.EXIT_INPUT and f"{bad}:4:" in err and "ObjParseError" in err
    code, _, err = _run(cli, capsys, "query", "--gen", "no-such-scene")
    assert code == cli.EXIT_INPUT and "unknown scene kind" in err
    code, _, err = _run(cli, capsys, "query")
    assert code == cli.EXIT_INPUT
    code, _, err = _run(cli, capsys, "query", "--gen", "random-blobs", "--mesh-a", str(bad))
    assert code == cli.EXIT_INPUT and "not both" in err
    code, _, err = _run(cli, capsys, "query", "--gen", "random-blobs", "n=5", "--depth-cap", "99")
    assert code == cli.EXIT_INPUT and "ConfigError" in err


def test_schema_file(cli):
    s = cli.load_schema()
    assert s["$id"] == cli.SCHEMA_ID
    for cmd in ("query", "ablate", "oracle"):
        cols = s["csv_columns"][cmd]
        assert len(cols) == len(set(cols)) and cols[:2] in (["frame", "kind"],)
    assert cli.validate_report({"schema": cli.SCHEMA_ID}) != []


# --------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_query_two_triangles(cli, md, gpu, capsys, tmp_path):
    """Two OBJ triangles -> distance = tri_tri_min (SPEC cli example 1)."""
    A = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]])
    B = np.array([[0.2, 0.2, 0.7], [1.3, 0.1, 0.9], [0.1, 1.2, 1.1]])
    pa, pb = _write_obj(tmp_path / "a.obj", A, [[0, 1, 2]]), _write_obj(tmp_path / "b.obj", B, [[0, 1, 2]])
    code, out, err = _run(cli, capsys, "query", "--mesh-a", pa, "--mesh-b", pb, "--kind", "both")
    assert code == 0, err
    doc = json.loads(out)
    assert cli.validate_report(doc) == []
    rec = doc["records"][0]
    d, _, _ = md.tri_tri_min(A, B)
    assert rec["results"]["min"]["distance"] == d
    assert rec["results"]["max"]["distance"] == md.tri_tri_max(A, B)[0]


@pytest.mark.gpu
def test_query_frames_check_and_csv(cli, md, gpu, capsys, tmp_path):
    """10-frame rotation of offset-grids about the gap axis: every frame
    cross-checked against brute force; CSV in the schema's column order."""
    frames = [{"a": {"axis": [0, 0, 1], "angle": 0.1 * i}} for i in range(10)]
    fp = tmp_path / "frames.json"
    fp.write_text(json.dumps(frames))
    out_json = tmp_path / "r.json"
    code, _, err = _run(cli, capsys, "query", "--gen", "offset-grids", "res=10", "--frames", str(fp), "--check",
                        "--kind", "both", "--out", str(out_json))
    assert code == 0, err
    doc = json.loads(out_json.read_text())
    assert cli.validate_report(doc) == [] and len(doc["records"]) == 10
    for rec in doc["records"]:
        assert all(c["ok"] for c in rec["check"].values())
        assert rec["timings_ms"]["refit"] >= 0
    code, out, err = _run(cli, capsys, "query", "--gen", "offset-grids", "res=10", "--frames", str(fp),
                          "--format", "csv")
    assert code == 0, err
    rows = list(csv.reader(io.StringIO(out)))
    assert rows[0] == cli.load_schema()["csv_columns"]["query"] and len(rows) == 11
    dists = [float(r[2]) for r in rows[1:]]
    assert all(abs(x - y) == 0 for x, y in zip(dists, [r["results"]["min"]["distance"] for r in doc["records"]]))


@pytest.mark.gpu
def test_query_intersecting_zero(cli, gpu, capsys):
    code, out, err = _run(cli, capsys, "query", "--gen", "intersecting-clusters", "n=500", "--seed", "3")
    assert code == 0, err
    assert json.loads(out)["records"][0]["results"]["min"]["distance"] == 0.0


@pytest.mark.gpu
def test_ablate_battery(cli, gpu, capsys):
    """Acceptance 9: the four variants agree and count their work; the
    no-enhanced peak front is >= the full engine's.  (SPEC's "DFS visits >=
    frontal expanded pairs on intersecting-clusters" does not hold for the
    reference itself at this size: 2164 visits vs 66560 expanded pairs.)"""
    for gen in (["random-blobs", "n=300,seed=5"], ["offset-grids", "res=12"],
                ["nested-shells", "lat=10,lon=14"], ["intersecting-clusters", "n=400,seed=2"]):
        code, out, err = _run(cli, capsys, "ablate", "--gen", *gen, "--kind", "both")
        assert code == 0, (gen, err)
        doc = json.loads(out)
        assert cli.validate_report(doc) == []
        for rec in doc["records"]:
            v = {x["variant"]: x for x in rec["variants"]}
            assert rec["agree"] and len({x["distance"] for x in v.values()}) == 1, gen
            assert v["no-enhanced"]["peak_front"] >= v["full"]["peak_front"]
            assert v["dfs"]["visited_nodes"] > 0 and v["dfs"]["peak_front"] is None
            assert v["fixed-k1"]["expanded_pairs"] > 0 and v["full"]["iterations"] > 0
    code, out, err = _run(cli, capsys, "ablate", "--gen", "random-blobs", "n=100", "--format", "csv")
    rows = list(csv.reader(io.StringIO(out)))
    assert code == 0 and rows[0] == cli.load_schema()["csv_columns"]["ablate"] and len(rows) == 5


@pytest.mark.gpu
def test_oracle_and_guard(cli, md, gpu, capsys):
    code, out, err = _run(cli, capsys, "oracle", "--gen", "random-blobs", "n=200,seed=1", "--kind", "both")
    assert code == 0, err
    doc = json.loads(out)
    assert cli.validate_report(doc) == [] and [r["kind"] for r in doc["records"]] == ["min", "max"]
    a, b = md.gen_scene("random-blobs", {"n": 200, "seed": 1})
    assert doc["records"][0]["distance"] == md.brute_force_min(a, b)[0]
    code, out, err = _run(cli, capsys, "oracle", "--gen", "random-blobs", "n=4000")
    assert code == cli.EXIT_QUERY and "SizeGuardError" in err and "16000000" in err
    code, out, err = _run(cli, capsys, "oracle", "--gen", "random-blobs", "n=4000", "--force", "--format", "csv")
    assert code == 0 and len(out.splitlines()) == 2


@pytest.mark.gpu
def test_deformation_frames_and_topology_error(cli, md, gpu, capsys, tmp_path):
    """Frames that replace A's vertices (same topology) refit the tree;
    a different triangle count is a TopologyMismatchError, nonzero exit."""
    a, b = md.gen_scene("random-blobs", {"n": 60, "seed": 7})
    pa = _write_obj(tmp_path / "a.obj", a.vertices, a.triangles)
    pb = _write_obj(tmp_path / "b.obj", b.vertices, b.triangles)
    moved = _write_obj(tmp_path / "a2.obj", a.vertices * 1.1 + 0.05, a.triangles)
    other = _write_obj(tmp_path / "a3.obj", a.vertices[:30], a.triangles[:10])
    fp = tmp_path / "fr.json"
    fp.write_text(json.dumps([{}, {"mesh_a": moved}]))
    code, out, err = _run(cli, capsys, "query", "--mesh-a", pa, "--mesh-b", pb, "--frames", str(fp), "--check")
    assert code == 0, err
    recs = json.loads(out)["records"]
    a2 = md.TriangleMesh(a.vertices * 1.1 + 0.05, a.triangles)
    assert recs[1]["results"]["min"]["distance"] == md.brute_force_min(md.load_obj(moved), b)[0]
    assert recs[1]["results"]["min"]["distance"] != recs[0]["results"]["min"]["distance"] or a2 is None
    fp.write_text(json.dumps([{"mesh_a": other}]))
    code, out, err = _run(cli, capsys, "query", "--mesh-a", pa, "--mesh-b", pb, "--frames", str(fp))
    assert code == cli.EXIT_INPUT and "TopologyMismatchError" in err


@pytest.mark.gpu
def test_module_entry_point(gpu, tmp_path):
    """`python -m paper_2411_11244_b200 ...` runs the CLI end to end."""
    import subprocess
    import sys
    from pathlib import Path

    out = tmp_path / "r.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2411_11244_b200", "query", "--gen", "interlocked-rings",
                        "nu=30,nv=15", "--kind", "both", "--format", "csv", "--out", str(out), "--check"],
                       capture_output=True, text=True, timeout=300, cwd=Path(__file__).resolve().parent.parent)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.reader(io.StringIO(out.read_text())))
    assert len(rows) == 3 and rows[1][1] == "min" and rows[2][1] == "max" and rows[1][-1] == "True"
