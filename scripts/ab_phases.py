"""A/B helper: NIPS (or --workload) sweep + per-kernel phase times for the current
environment, one JSON line (used with env knobs on the GPU box)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
wl = sys.argv[1] if len(sys.argv) > 1 else "nips"
steps = sys.argv[2] if len(sys.argv) > 2 else "20"
r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--steps", steps,
                    "--warmup", "5", "--no-cpu-baseline"], capture_output=True, text=True)
try:
    d = json.loads(r.stdout.strip().splitlines()[-1])
    keys = {k: v for k, v in os.environ.items() if k.startswith("BNMC_")}
    print(json.dumps({"env": keys, "wl": wl, "ms": round(d["ms_per_step"], 5), "phases": d.get("phases_ms"),
                      "e2e_ms": (d.get("e2e") or {}).get("ms_per_step"), "lj": d.get("last_log_joint"),
                      "sm_mhz": d["clocks"]["sm_mhz"]}))
except Exception as e:  # noqa: BLE001
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("BNMC_")}, "error": str(e),
                      "stderr": r.stderr[-800:]}))
