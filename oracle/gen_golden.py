"""Generate golden fixtures from the REAL reference (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py [--ref /root/reference/pkg/src]

Imports `modelmerge` from the read-only reference tree and records, with
fixed seeds, (a) kernel input/output vectors for every engine kernel,
(b) the merged-graph structure the reference emits for each zoo model and
model count, and (c) merged-execution outputs per model for the zoo
verify matrix. Outputs go to tests/golden/ and are committed; the GPU box
never needs the reference. TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"


def _rand(rng, shape, dtype, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, size=shape).astype(dtype)


def kernel_vectors(E, MergeDim):
    """Seeded kernel calls; arrays stored as key -> array in one npz."""
    rng = np.random.default_rng(20261017)
    rec: dict[str, np.ndarray] = {}
    meta: list[dict] = []

    def put(name, fn, args, kwargs, arrays):
        out = fn(*args, **kwargs)
        for i, a in enumerate(arrays):
            rec[f"{name}/in{i}"] = a
        if isinstance(out, list):
            for i, o in enumerate(out):
                rec[f"{name}/out{i}"] = o
            nout = len(out)
        else:
            rec[f"{name}/out0"] = out
            nout = 1
        meta.append({"name": name, "fn": fn.__name__, "n_in": len(arrays), "n_out": nout,
                     "kwargs": {k: (v.value if hasattr(v, "value") else v)
                                for k, v in kwargs.items()}})

    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        for (k, s, p) in [(1, 1, 0), (3, 1, 1), (3, 2, 1), (7, 2, 3), (1, 2, 0)]:
            x, w, b = _rand(rng, (2, 3, 9, 9), dt), _rand(rng, (4, 3, k, k), dt, -.5, .5), \
                _rand(rng, (4,), dt, -.5, .5)
            put(f"conv2d_{tag}_k{k}s{s}p{p}", E.conv2d, (x, w, b), {"stride": s, "padding": p},
                [x, w, b])
        for g, cin, cout in [(2, 4, 6), (4, 8, 8), (3, 3, 6), (8, 32, 16)]:
            x = _rand(rng, (2, cin, 8, 8), dt)
            w = _rand(rng, (cout, cin // g, 3, 3), dt, -.5, .5)
            b = _rand(rng, (cout,), dt, -.5, .5)
            put(f"gconv_{tag}_g{g}_{cin}_{cout}", E.grouped_conv2d, (x, w, b),
                {"groups": g, "stride": 1, "padding": 1}, [x, w, b])
        x, w, b = _rand(rng, (3, 5, 12), dt), _rand(rng, (12, 7), dt, -.5, .5), \
            _rand(rng, (7,), dt, -.5, .5)
        put(f"matmul_{tag}", E.matmul, (x, w, b), {}, [x, w, b])
        x, w, b = _rand(rng, (4, 6, 24), dt), _rand(rng, (4, 24, 10), dt, -.5, .5), \
            _rand(rng, (4, 10), dt, -.5, .5)
        put(f"bmm3_{tag}", E.batch_matmul, (x, w, b), {}, [x, w, b])
        x, w = _rand(rng, (3, 2, 5, 16), dt), _rand(rng, (3, 16, 8), dt, -.5, .5)
        put(f"bmm4_{tag}", E.batch_matmul, (x, w), {}, [x, w])
        for shape in [(4, 16), (2, 5, 24), (2, 8, 3, 3)]:
            c = shape[1 if len(shape) != 3 else 2]
            x, g_, b_ = _rand(rng, shape, dt), _rand(rng, (c,), dt, .5, 1.5), \
                _rand(rng, (c,), dt, -.5, .5)
            put(f"ln_{tag}_r{len(shape)}", E.layer_norm, (x, g_, b_), {"eps": 1e-5}, [x, g_, b_])
            put(f"gn_{tag}_r{len(shape)}", E.group_norm, (x, g_, b_), {"groups": 4, "eps": 1e-5},
                [x, g_, b_])
        x = _rand(rng, (2, 6, 5, 5), dt)
        vecs = [_rand(rng, (6,), dt) for _ in range(3)] + [_rand(rng, (6,), dt, .5, 1.5)]
        put(f"bn_{tag}", E.batch_norm_inference, (x, *vecs), {"eps": 1e-5}, [x, *vecs])
        x = _rand(rng, (3, 7, 9), dt, -4, 4)
        put(f"relu_{tag}", E.relu, (x,), {}, [x])
        put(f"tanh_{tag}", E.tanh, (x,), {}, [x])
        for ax in (-1, 1, 0):
            put(f"softmax_{tag}_ax{ax}", E.softmax, (x,), {"axis": ax}, [x])
        y = _rand(rng, (3, 7, 9), dt)
        put(f"add_{tag}", E.add, (x, y), {}, [x, y])
        put(f"mul_{tag}", E.mul, (x, y), {}, [x, y])
        x = _rand(rng, (2, 3, 8, 8), dt)
        put(f"maxpool_{tag}_k2", E.max_pool2d, (x,), {"kernel": 2, "stride": 2}, [x])
        put(f"maxpool_{tag}_k3s1", E.max_pool2d, (x,), {"kernel": 3, "stride": 1}, [x])
        put(f"meanpool_{tag}_k2", E.mean_pool2d, (x,), {"kernel": 2, "stride": 2}, [x])
        put(f"meanpool_{tag}_k8", E.mean_pool2d, (x,), {"kernel": 8, "stride": 8}, [x])
    # known-answer vectors from the reference's own tests (test_engine_core.py:136-144)
    x = np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4)
    put("maxpool_kat", E.max_pool2d, (x,), {"kernel": 2, "stride": 2}, [x])
    put("meanpool_kat", E.mean_pool2d, (x,), {"kernel": 2, "stride": 2}, [x])
    # pack / unpack round trips
    for dim in ("channel", "batch"):
        for shape in [(2, 4), (2, 3, 4), (2, 4, 3, 3)]:
            parts = [_rand(rng, shape, np.float32) for _ in range(3)]
            d = MergeDim(dim)
            put(f"pack_{dim}_r{len(shape)}", lambda *ps, dim=d: E.pack(list(ps), dim=dim),
                tuple(parts), {}, parts)
    return rec, meta


def _graph_doc(graph, layout_attr=True):
    return {
        "nodes": [{"id": n.id, "kind": n.kind.value, "inputs": list(n.inputs),
                   "weights": list(n.weights), "attrs": n.attrs,
                   "dims": list(n.output_spec.dims), "dtype": n.output_spec.dtype,
                   "layout": n.output_spec.layout.value} for n in graph.nodes],
        "graph_inputs": {k: {"dims": list(v.dims), "dtype": v.dtype, "layout": v.layout.value}
                         for k, v in graph.graph_inputs.items()},
        "graph_outputs": list(graph.graph_outputs),
    }


def merge_structures(mm):
    docs = {}
    for name in ("ffnn", "cnnblock", "attnblock"):
        for m in (1, 2, 3, 4):
            for batch in (1, 2):
                graph, stores = mm.build_zoo(name, num_models=m, batch=batch)
                merged, _ = mm.merge(graph, stores)
                docs[f"{name}/m{m}/b{batch}"] = {
                    "source": _graph_doc(graph),
                    "merged": _graph_doc(merged.graph),
                    "node_dims": {k: v.value for k, v in merged.node_dims.items()},
                    "glue": [{"index": g.index, "producer": g.producer, "src": g.src_dim.value,
                              "dst": g.dst_dim.value, "nodes": list(g.node_ids)}
                             for g in merged.glue],
                    "input_plan": merged.input_plan,
                    "output_plan": merged.output_plan,
                    "dispatch_count": merged.dispatch_count,
                    "node_visits": merged.stats.node_visits,
                    "edge_inspections": merged.stats.edge_inspections,
                    "explain": mm.explain(merged),
                }
    return docs


def zoo_outputs(mm):
    """Reference merged execution per (model, M, B, dtype): weights/inputs are
    regenerated by the zoo's seeding; outputs and a weight checksum stored."""
    rec = {}
    for name in ("ffnn", "cnnblock", "attnblock"):
        for m in (1, 2, 4):
            for batch in (1, 4):
                for dtype in ("f32", "f64"):
                    graph, stores = mm.build_zoo(name, num_models=m, batch=batch, dtype=dtype)
                    inputs = [mm.model_inputs(graph, seed=0, model=j) for j in range(m)]
                    merged, mstore = mm.merge(graph, stores)
                    outs, _ = mm.execute(merged.graph, mstore, merged.bind_inputs(inputs))
                    per = merged.slice_outputs(outs)
                    key = f"{name}/m{m}/b{batch}/{dtype}"
                    for j in range(m):
                        rec[f"{key}/out{j}"] = per[j][0].data
                        solo, _ = mm.execute(graph, stores[j], inputs[j])
                        assert solo[0].bit_equal(per[j][0])
                    rec[f"{key}/wsum"] = np.array(
                        [sum(float(np.sum(t.data, dtype=np.float64)) for t in s.tensors.values())
                         for s in stores])
    return rec


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args(argv)
    sys.path.insert(0, args.ref)
    sys.dont_write_bytecode = True
    # The reference's package __init__ pulls in the CLI/plotting stack
    # (matplotlib, absent here); import the submodules we need directly.
    import importlib
    import types
    pkg = types.ModuleType("modelmerge")
    pkg.__path__ = [str(Path(args.ref) / "modelmerge")]
    sys.modules["modelmerge"] = pkg
    E = importlib.import_module("modelmerge.engine")
    ir = importlib.import_module("modelmerge.ir")
    merger = importlib.import_module("modelmerge.merger")
    zoo = importlib.import_module("modelmerge.zoo")

    class MM:
        build_zoo = staticmethod(zoo.build_zoo)
        model_inputs = staticmethod(zoo.model_inputs)
        merge = staticmethod(merger.merge)
        explain = staticmethod(merger.explain)
        execute = staticmethod(E.execute)

    OUT.mkdir(parents=True, exist_ok=True)
    rec, meta = kernel_vectors(E, ir.MergeDim)
    np.savez_compressed(OUT / "kernels.npz", **rec)
    (OUT / "kernels.json").write_text(json.dumps(meta, indent=1) + "\n")
    (OUT / "merge_structures.json").write_text(json.dumps(merge_structures(MM), indent=1) + "\n")
    np.savez_compressed(OUT / "zoo_outputs.npz", **zoo_outputs(MM))
    golden = Path(args.ref).parent / "tests" / "data" / "ffnn_m2_golden.json"
    if golden.exists():  # cross-check: our structure dump agrees with the reference golden
        ref_doc = json.loads(golden.read_text())
        ours = json.loads((OUT / "merge_structures.json").read_text())["ffnn/m2/b1"]["merged"]
        assert [n["id"] for n in ref_doc["nodes"]] == [n["id"] for n in ours["nodes"]]
    print("wrote", sorted(p.name for p in OUT.iterdir()))
    return 0


if __name__ == "__main__":
    sys.exit(main())
