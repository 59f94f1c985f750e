"""Golden artifact fixtures from the REAL reference serializer (run in the
build container; the GPU box never needs the reference). TEST
INFRASTRUCTURE ONLY.

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_artifacts.py [--ref /root/reference/pkg/src]

Writes tests/golden/artifacts/: the reference's merged ffnn (M=2) and
cnnblock (M=3) graphs with embedded merge records (``serialize``,
serialize.py:53-77), and TNSR blobs of seeded f32 / f64 tensors
(``tensor_to_bytes``, serialize.py:168-175), plus a store directory
(``save_weight_store``, serialize.py:220-234) of the merged ffnn weights.
"""

from __future__ import annotations

import argparse
import importlib
import json
import shutil
import sys
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "artifacts"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args(argv)
    sys.path.insert(0, args.ref)
    sys.dont_write_bytecode = True
    pkg = types.ModuleType("modelmerge")  # skip the CLI/plotting __init__ (matplotlib)
    pkg.__path__ = [str(Path(args.ref) / "modelmerge")]
    sys.modules["modelmerge"] = pkg
    E = importlib.import_module("modelmerge.engine")
    ir = importlib.import_module("modelmerge.ir")
    merger = importlib.import_module("modelmerge.merger")
    zoo = importlib.import_module("modelmerge.zoo")
    ser = importlib.import_module("modelmerge.serialize")

    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    for name, m in (("ffnn", 2), ("cnnblock", 3)):
        graph, stores = zoo.build_zoo(name, num_models=m)
        merged, mstore = merger.merge(graph, stores)
        merged.embed_metadata()
        (OUT / f"{name}_m{m}.json").write_bytes(ser.serialize(merged.graph))
        if name == "ffnn":
            ser.save_weight_store(mstore, OUT / "ffnn_m2_store")
    rng = np.random.default_rng(20261017)
    cases = {}
    for i, (dtype, dims) in enumerate((("f32", (3, 5)), ("f64", (2, 3, 4)), ("f32", (7,)))):
        arr = rng.uniform(-2, 2, dims).astype(np.float32 if dtype == "f32" else np.float64)
        tv = E.TensorValue(ir.TensorSpec(dtype, dims), arr)
        (OUT / f"t{i}.tnsr").write_bytes(ser.tensor_to_bytes(tv))
        np.save(OUT / f"t{i}.npy", arr)
        cases[f"t{i}"] = {"dtype": dtype, "dims": list(dims)}
    (OUT / "tensors.json").write_text(json.dumps(cases, indent=1) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))
    return 0


if __name__ == "__main__":
    sys.exit(main())
