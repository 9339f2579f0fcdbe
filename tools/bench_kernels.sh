#!/bin/bash
# per-kernel ms/step of a short bench run (for A/B experiments); usage: tools/bench_kernels.sh [bench args]
python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" 2>/dev/null | python tools/bench_summary.py
