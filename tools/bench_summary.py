"""Print a compact summary of bench.py JSON line(s) read from stdin or a file (diagnostics)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
for line in src:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "kernels" not in d:
        print(line[:300])
        continue
    k = {n: round(v["ms_per_step"], 1) for n, v in d["kernels"].items()}
    print(f"value={d['value']:.0f} {d['unit']} ms/step={d['ms_per_step']:.1f} roofline={d['roofline']['frac']:.3f} "
          f"e2e={d['e2e']['value']:.0f} clocks={d.get('clocks')}\n  kernels={k}\n"
          f"  merge_output_error={(d.get('merge_output_error') or {}).get('value')}\n"
          f"  stale_profiling={d.get('stale_profiling')}")
