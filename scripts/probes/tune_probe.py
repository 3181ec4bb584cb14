"""Run the GPU autotuner (verify-before-time over every tcgen05 config x split) on shapes where
the planner's choice trails cuBLASLt, and print the winner next to the planner's default."""
import json
import sys

sys.path.insert(0, ".")
from paper_1910_00178_b200 import api  # noqa: E402

for sh in sys.argv[1:] or ["2048x2048x2048", "4096x4096x4096", "2048x4096x1024"]:
    m, n, k = (int(x) for x in sh.split("x"))
    r = api.tune(m, n, k, api.SatMode.WIDENING_EXACT, repeats=21, warmup=5)
    print(json.dumps({"shape": sh, **{kk: (round(v, 1) if isinstance(v, float) else v) for kk, v in r.items()}}), flush=True)
