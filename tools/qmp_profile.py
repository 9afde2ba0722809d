"""Runs bench.py's qmp_nonfactorised variant alone (for an ncu launch list of the Q_MP row's kernels)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

print(json.dumps(bench.run_qmp_variant("cuda:0", steps=2)))
