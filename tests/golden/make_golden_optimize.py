"""Golden optimizer traces from the REFERENCE (run in the build container):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_optimize.py
Writes golden_optimize.json (histories of the reference's Nelder-Mead)."""

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from qaoa_maxcut import random_regular_graph  # noqa: E402
from qaoa_maxcut.optimize import optimize  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
runs = []
for n, p, budget, init, seed in ((10, 2, 120, "linear-ramp", 0), (8, 1, 60, "random", 3),
                                 (12, 3, 80, "linear-ramp", 1)):
    g = random_regular_graph(n, 3, seed=seed)
    rep = optimize(g, p=p, backend="bitwise", budget=budget, seed=seed, init_strategy=init)
    runs.append({"n": n, "p": p, "budget": budget, "init": init, "seed": seed,
                 "report": rep.to_dict()})
with open(os.path.join(HERE, "golden_optimize.json"), "w") as f:
    json.dump(runs, f)
print("wrote", len(runs))
