"""Time batched private inference (bench.ppml_rates) at a few batch sizes.

    python tools/ppml_probe.py mlp 256:16 4096:64
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402
import bench  # noqa: E402

name = sys.argv[1]
for spec in sys.argv[2:]:
    b, vb = (int(x) for x in spec.split(":"))
    print(json.dumps(bench.ppml_rates(name, b, vb)), flush=True)
