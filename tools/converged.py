"""Converged-regime timing only (bench.run_converged_variant), one JSON line per config."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

out = bench.run_converged_variant(None, torch.device("cuda:0"))
for k, v in out.items():
    print(k, round(v["ms_per_step"], 3), "fwd", round(v["forward_ms"], 3), v["forward_mode_hist"],
          v["forward_roofline"].get("frac", v["forward_roofline"].get("over_pairwise_ceiling")), "bwd moment groups", v["backward_moment_groups"])
