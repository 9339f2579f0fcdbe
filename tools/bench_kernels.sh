#!/bin/bash
# per-kernel ms/step of a short bench run (for A/B experiments); usage: tools/bench_kernels.sh [bench args]
python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(round(d['value']), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items() if k.startswith('gemm')}, d['clocks']['sm_mhz'] if d['clocks'] else None)"
