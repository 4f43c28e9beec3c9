"""Command-line front end (SPEC.md [MODULE] cli).

    python -m paper_2411_11244_b200 query  --gen interlocked-rings nu=100,nv=50 --kind both
    python -m paper_2411_11244_b200 ablate --mesh-a a.obj --mesh-b b.obj --kind min
    python -m paper_2411_11244_b200 oracle --gen random-blobs n=200 --force --format csv

* query  -- build both trees once, then per frame: refit, the requested
  queries, one report record (QueryResult JSON + build / refit / query
  wall-clock ms).  `--check` cross-checks every frame with the device brute
  force (test mode: exit 4 on a mismatch).
* ablate -- the paper's ablation (section 8.2): full engine, enhanced bounds
  off (gDist-v1), fixed k = 1 (gDist-v2) and the per-triangle DFS comparator
  (query.py:622-708); all four distances must agree (exit 4 otherwise).
* oracle -- brute force (query.py:571-619), size guard unless --force.

Frames (`--frames FILE`, JSON): either a list whose elements are
{"a": XF, "b": XF, "mesh_a": OBJ, "mesh_b": OBJ} (every key optional; a bare
XF applies to A) or an object {"a": [XF, ...], "b": [XF, ...]} of equal
lengths.  XF = {"rotation": 3x3, "translation": [3]} or {"axis": [3],
"angle": radians, "translation": [3]} or null.  "mesh_a"/"mesh_b" replace the
mesh's vertices for that frame (deformation: same triangle count, else the
refit raises TopologyMismatchError).

Reports follow report_schema.json (JSON: one document with a record per frame;
CSV: the schema's fixed column order, one row per frame and query kind).
Exit codes: 0 ok, 2 input / usage error, 3 query failure, 4 cross-check
failure.  The device path is the only path: no GPU -> exit 3.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

EXIT_OK, EXIT_INPUT, EXIT_QUERY, EXIT_CHECK = 0, 2, 3, 4
SCHEMA_ID = "gdist-report/1"
SCHEMA_PATH = Path(__file__).with_name("report_schema.json")


class CliError(Exception):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(message)


# ---------------------------------------------------------------------------
# argument parsing
# ---------------------------------------------------------------------------
def _scalar(text: str):
    low = text.lower()
    if low in ("true", "false"):
        return low == "true"
    for conv in (int, float):
        try:
            return conv(text)
        except ValueError:
            pass
    return text


def parse_gen_params(text: str | None) -> dict:
    """'k=v,k2=v2' -> {k: v}; values int, float, bool or string; a value in
    brackets is a comma-free tuple ('center=[0;0;1]' -> (0, 0, 1))."""
    out = {}
    if not text:
        return out
    for item in text.split(","):
        item = item.strip()
        if not item:
            continue
        if "=" not in item:
            raise CliError(EXIT_INPUT, f"--gen parameter {item!r} is not k=v")
        k, v = item.split("=", 1)
        v = v.strip()
        if v.startswith("[") and v.endswith("]"):
            out[k.strip()] = tuple(_scalar(x) for x in v[1:-1].split(";") if x.strip())
        else:
            out[k.strip()] = _scalar(v)
    return out


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2411_11244_b200",
                                description="Exact min / max distance between triangle meshes on B200.")
    p.add_argument("command", choices=("query", "ablate", "oracle"))
    p.add_argument("--mesh-a", metavar="PATH")
    p.add_argument("--mesh-b", metavar="PATH")
    p.add_argument("--gen", nargs="+", metavar=("KIND", "K=V,..."), help="scene generator and its parameters")
    p.add_argument("--kind", choices=("min", "max", "both"), default="min")
    p.add_argument("--frames", metavar="FILE")
    p.add_argument("--precision", type=int, choices=(32, 64), default=64)
    p.add_argument("--front-cap", type=int, default=262_144)
    p.add_argument("--depth-cap", type=int, default=5)
    p.add_argument("--no-enhanced", action="store_true")
    p.add_argument("--threads", default=os.environ.get("MESHDIST_THREADS", "1"),
                   help="accepted for compatibility (the device engine ignores it); default $MESHDIST_THREADS")
    p.add_argument("--seed", type=int)
    p.add_argument("--out", default="-", metavar="PATH")
    p.add_argument("--format", choices=("json", "csv"), default="json")
    p.add_argument("--force", action="store_true", help="lift the brute-force size guard")
    p.add_argument("--check", action="store_true", help="test mode: cross-check every result with brute force")
    return p


def engine_config(args):
    from .query import EngineConfig

    threads = args.threads if args.threads == "auto" else int(args.threads)
    return EngineConfig(front_cap=args.front_cap, depth_cap=args.depth_cap, precision=args.precision,
                        threads=threads, enhanced_bounds=not args.no_enhanced)


def load_inputs(args):
    """(mesh_a, mesh_b, description): exactly one source per mesh."""
    from .mesh import load_obj
    from .scenes import _GENERATORS, gen_scene

    if args.gen and (args.mesh_a or args.mesh_b):
        raise CliError(EXIT_INPUT, "give either --gen or --mesh-a/--mesh-b, not both")
    if args.gen:
        if len(args.gen) > 2:
            raise CliError(EXIT_INPUT, "--gen takes KIND and one k=v,... list")
        kind = args.gen[0]
        params = parse_gen_params(args.gen[1] if len(args.gen) > 1 else None)
        gen = _GENERATORS.get(kind)
        if args.seed is not None and gen is not None and "seed" in gen.__code__.co_varnames and "seed" not in params:
            params["seed"] = args.seed
        a, b = gen_scene(kind, params)
        return a, b, {"gen": kind, "params": {k: list(v) if isinstance(v, tuple) else v for k, v in params.items()}}
    if not (args.mesh_a and args.mesh_b):
        raise CliError(EXIT_INPUT, "need --gen KIND or both --mesh-a and --mesh-b")
    return load_obj(args.mesh_a), load_obj(args.mesh_b), {"mesh_a": args.mesh_a, "mesh_b": args.mesh_b}


def _xf(obj, where: str):
    from .mesh import RigidTransform

    if obj is None:
        return None
    if not isinstance(obj, dict):
        raise CliError(EXIT_INPUT, f"{where}: a transform is an object, got {type(obj).__name__}")
    t = obj.get("translation", (0.0, 0.0, 0.0))
    try:
        if "rotation" in obj:
            return RigidTransform(obj["rotation"], t)
        if "axis" in obj:
            return RigidTransform.from_axis_angle(obj["axis"], float(obj.get("angle", 0.0)), t)
        return RigidTransform(None, t)
    except (ValueError, TypeError) as exc:
        raise CliError(EXIT_INPUT, f"{where}: {exc}") from None


def load_frames(path: str | None) -> list:
    """-> [(xf_a, xf_b, obj_a, obj_b)] (None = unchanged); [] = one frame, no motion."""
    if not path:
        return []
    try:
        data = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise CliError(EXIT_INPUT, f"--frames {path}: {exc}") from None
    frames = []
    if isinstance(data, dict):
        fa, fb = data.get("a"), data.get("b")
        if fa is not None and fb is not None and len(fa) != len(fb):
            raise CliError(EXIT_INPUT, f"--frames {path}: {len(fa)} transforms for A but {len(fb)} for B")
        n = len(fa if fa is not None else fb or [])
        for i in range(n):
            frames.append((_xf(fa[i], f"frame {i} a") if fa is not None else None,
                           _xf(fb[i], f"frame {i} b") if fb is not None else None, None, None))
    elif isinstance(data, list):
        for i, el in enumerate(data):
            if isinstance(el, dict) and ({"a", "b", "mesh_a", "mesh_b"} & set(el)):
                frames.append((_xf(el.get("a"), f"frame {i} a"), _xf(el.get("b"), f"frame {i} b"),
                               el.get("mesh_a"), el.get("mesh_b")))
            else:
                frames.append((_xf(el, f"frame {i}"), None, None, None))
    else:
        raise CliError(EXIT_INPUT, f"--frames {path}: expected a JSON list or object")
    return frames


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------
def _sync():
    from . import _lib

    _lib.torch().cuda.synchronize()


def _frame_meshes(base_a, base_b, frame, cache):
    """The meshes of one frame: deformation (OBJ) first, then the transform."""
    from .mesh import TriangleMesh, apply_transform, load_obj

    if frame is None:
        return base_a, base_b
    xa, xb, oa, ob = frame
    out = []
    for base, xf, obj in ((base_a, xa, oa), (base_b, xb, ob)):
        m = base
        if obj is not None:
            if obj not in cache:
                cache[obj] = load_obj(obj)
            d = cache[obj]
            # deformation: the file's vertices on this mesh's connectivity
            m = TriangleMesh(d.vertices, d.triangles)
        if xf is not None:
            m = apply_transform(m, xf)
        out.append(m)
    return out[0], out[1]


def _kinds(args):
    return ("min", "max") if args.kind == "both" else (args.kind,)


def _brute(a, b, kind, args, dtype):
    from .query import brute_force_max, brute_force_min

    return (brute_force_min if kind == "min" else brute_force_max)(a, b, force=args.force, dtype=dtype)


def cmd_query(args, base_a, base_b, frames, cfg) -> tuple[list, bool]:
    from .bvh import build_f12, refit
    from .query import run_max_query, run_min_query

    t0 = time.perf_counter()
    bvh_a, bvh_b = build_f12(base_a, dtype=cfg.dtype), build_f12(base_b, dtype=cfg.dtype)
    _sync()
    build_ms = (time.perf_counter() - t0) * 1e3
    records, ok, cache = [], True, {}
    for f, frame in enumerate(frames or [None]):
        a, b = _frame_meshes(base_a, base_b, frame, cache)
        t0 = time.perf_counter()
        refit(bvh_a, a)
        refit(bvh_b, b)
        _sync()
        refit_ms = (time.perf_counter() - t0) * 1e3
        results, q_ms, checks = {}, {}, {}
        for kind in _kinds(args):
            t0 = time.perf_counter()
            r = (run_min_query if kind == "min" else run_max_query)(a, b, bvh_a, bvh_b, cfg)
            q_ms[kind] = (time.perf_counter() - t0) * 1e3
            results[kind] = r.to_json_dict()
            if args.check:
                d, w = _brute(a, b, kind, args, cfg.dtype)
                good = d == r.distance
                ok &= good
                checks[kind] = {"brute_distance": d, "brute_tri_a": w.tri_a, "brute_tri_b": w.tri_b, "ok": good}
        rec = {"frame": f, "n_tris_a": a.n_triangles, "n_tris_b": b.n_triangles, "results": results,
               "timings_ms": {"build": build_ms if f == 0 else 0.0, "refit": refit_ms, "query": q_ms}}
        if args.check:
            rec["check"] = checks
        records.append(rec)
    return records, ok


def cmd_ablate(args, base_a, base_b, frames, cfg) -> tuple[list, bool]:
    from .bvh import build_f12, refit
    from .query import run_dfs_baseline, run_max_query, run_min_query

    variants = [("full", cfg), ("no-enhanced", replace(cfg, enhanced_bounds=False)),
                ("fixed-k1", replace(cfg, depth_cap=1)), ("dfs", None)]
    bvh_a, bvh_b = build_f12(base_a, dtype=cfg.dtype), build_f12(base_b, dtype=cfg.dtype)
    records, ok, cache = [], True, {}
    for f, frame in enumerate(frames or [None]):
        a, b = _frame_meshes(base_a, base_b, frame, cache)
        refit(bvh_a, a)
        refit(bvh_b, b)
        for kind in _kinds(args):
            rows = []
            for name, vcfg in variants:
                _sync()
                t0 = time.perf_counter()
                if vcfg is None:
                    r = run_dfs_baseline(a, b, bvh_b, kind)
                else:
                    r = (run_min_query if kind == "min" else run_max_query)(a, b, bvh_a, bvh_b, vcfg)
                ms = (time.perf_counter() - t0) * 1e3
                rows.append({"variant": name, "distance": r.distance,
                             "tri_a": None if r.witness is None else r.witness.tri_a,
                             "tri_b": None if r.witness is None else r.witness.tri_b,
                             "expanded_pairs": r.expanded_pairs, "visited_nodes": r.visited_nodes,
                             "narrow_pairs": r.narrow_pairs,
                             "peak_front": None if vcfg is None else r.peak_front,
                             "iterations": len(r.iterations), "time_ms": ms})
            # the DFS comparator evaluates in float64 (as the reference's);
            # it joins the agreement check when the engine does too
            compared = [x["distance"] for x in rows if x["variant"] != "dfs" or cfg.precision == 64]
            agree = all(d == compared[0] for d in compared)
            ok &= agree
            records.append({"frame": f, "kind": kind, "agree": agree, "variants": rows})
    return records, ok


def cmd_oracle(args, base_a, base_b, frames, cfg) -> tuple[list, bool]:
    records, cache = [], {}
    for f, frame in enumerate(frames or [None]):
        a, b = _frame_meshes(base_a, base_b, frame, cache)
        for kind in _kinds(args):
            t0 = time.perf_counter()
            d, w = _brute(a, b, kind, args, cfg.dtype)
            ms = (time.perf_counter() - t0) * 1e3
            records.append({"frame": f, "kind": kind, "distance": d, "tri_a": w.tri_a, "tri_b": w.tri_b,
                            "point_a": [float(x) for x in w.point_a], "point_b": [float(x) for x in w.point_b],
                            "pairs": a.n_triangles * b.n_triangles, "time_ms": ms})
    return records, True


COMMANDS = {"query": cmd_query, "ablate": cmd_ablate, "oracle": cmd_oracle}


# ---------------------------------------------------------------------------
# reports
# ---------------------------------------------------------------------------
def load_schema() -> dict:
    return json.loads(SCHEMA_PATH.read_text())


def validate_report(doc: dict) -> list:
    """Problems of a JSON report against report_schema.json's required keys
    (no third-party validator in the image); [] = valid."""
    schema = load_schema()
    errs = [f"missing top-level key {k!r}" for k in schema["required"] if k not in doc]
    if errs:
        return errs
    if doc["schema"] != SCHEMA_ID:
        errs.append(f"schema id {doc['schema']!r} != {SCHEMA_ID!r}")
    cmd = doc["command"]
    if cmd not in schema["records"]:
        return errs + [f"unknown command {cmd!r}"]
    errs += [f"config lacks {k!r}" for k in schema["properties"]["config"]["required"] if k not in doc["config"]]
    rec_req = schema["records"][cmd]["required"]
    for i, rec in enumerate(doc["records"]):
        errs += [f"record {i} lacks {k!r}" for k in rec_req if k not in rec]
        if cmd == "query":
            for kind, r in rec.get("results", {}).items():
                errs += [f"record {i} {kind} result lacks {k!r}" for k in schema["query_result"]["required"]
                         if k not in r]
        elif cmd == "ablate":
            req = schema["records"]["ablate"]["properties"]["variants"]["items"]["required"]
            for v in rec.get("variants", []):
                errs += [f"record {i} variant lacks {k!r}" for k in req if k not in v]
    return errs


def csv_rows(command: str, records: list) -> tuple[list, list]:
    """Flatten records into the schema's fixed column order."""
    cols = load_schema()["csv_columns"][command]
    rows = []
    for rec in records:
        if command == "query":
            for kind, r in rec["results"].items():
                pa, pb = r["point_a"] or [None] * 3, r["point_b"] or [None] * 3
                chk = rec.get("check", {}).get(kind, {})
                vals = {"frame": rec["frame"], "kind": kind, "distance": r["distance"],
                        "witness_exact": r["witness_exact"], "tri_a": r["tri_a"], "tri_b": r["tri_b"],
                        "point_a_x": pa[0], "point_a_y": pa[1], "point_a_z": pa[2],
                        "point_b_x": pb[0], "point_b_y": pb[1], "point_b_z": pb[2],
                        "iterations": len(r["iterations"]), "expanded_pairs": r["expanded_pairs"],
                        "narrow_pairs": r["narrow_pairs"], "peak_front": r["peak_front"],
                        "build_ms": rec["timings_ms"]["build"], "refit_ms": rec["timings_ms"]["refit"],
                        "query_ms": rec["timings_ms"]["query"][kind], "check_ok": chk.get("ok")}
                rows.append([vals[c] for c in cols])
        elif command == "ablate":
            for v in rec["variants"]:
                vals = dict(v, frame=rec["frame"], kind=rec["kind"], agree=rec["agree"])
                rows.append([vals[c] for c in cols])
        else:
            vals = dict(rec)
            for side in ("a", "b"):
                for i, ax in enumerate("xyz"):
                    vals[f"point_{side}_{ax}"] = rec[f"point_{side}"][i]
            rows.append([vals[c] for c in cols])
    return cols, rows


def render(command: str, args, inputs: dict, cfg, records: list) -> str:
    if args.format == "csv":
        cols, rows = csv_rows(command, records)
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(cols)
        w.writerows(["" if x is None else x for x in row] for row in rows)
        return buf.getvalue()
    doc = {"schema": SCHEMA_ID, "command": command, "inputs": inputs,
           "config": {"kind": args.kind, "precision": cfg.precision, "front_cap": cfg.front_cap,
                      "depth_cap": cfg.depth_cap, "enhanced_bounds": cfg.enhanced_bounds,
                      "threads": cfg.threads, "force": bool(args.force), "check": bool(args.check)},
           "records": records}
    return json.dumps(doc, indent=1, allow_nan=True) + "\n"


def main(argv=None) -> int:
    from .errors import (ConfigError, FrontOverflowError, MeshDistError, ObjParseError, SceneError,
                         SizeGuardError, TopologyMismatchError)

    args = build_parser().parse_args(argv)
    try:
        try:
            cfg = engine_config(args)
            a, b, inputs = load_inputs(args)
            frames = load_frames(args.frames)
        except (ObjParseError, SceneError, ConfigError, ValueError, OSError) as exc:
            raise CliError(EXIT_INPUT, f"{type(exc).__name__}: {exc}") from None
        try:
            records, ok = COMMANDS[args.command](args, a, b, frames, cfg)
        except (TopologyMismatchError, ObjParseError, ConfigError) as exc:
            raise CliError(EXIT_INPUT, f"{type(exc).__name__}: {exc}") from None
        except (FrontOverflowError, SizeGuardError, MeshDistError, RuntimeError) as exc:
            raise CliError(EXIT_QUERY, f"{type(exc).__name__}: {exc}") from None
        text = render(args.command, args, inputs, cfg, records)
        if args.out == "-":
            sys.stdout.write(text)
        else:
            Path(args.out).write_text(text)
        if not ok:
            print("error: cross-check failed (distances disagree)", file=sys.stderr)
            return EXIT_CHECK
        return EXIT_OK
    except CliError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return exc.code


if __name__ == "__main__":
    sys.exit(main())
