"""Summarise one bench JSON line from stdin: tag, value, ms/step, SM clock, per-stage us (--detail)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
st = {k: v["us"] for k, v in (d.get("stages") or {}).items()}
print(sys.argv[1] if len(sys.argv) > 1 else "", d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], json.dumps(st))
