python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for i in 1 2; do
for c in off on; do
  timeout 400 python bench.py --other-configs "" --rounds 0 --error-tokens 0 --no-cpu-baseline --chain $c > gpurun_out/ab_ds_${c}_$i.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/ab_ds_${c}_$i.log") if x.startswith("{")][-1]; d=json.loads(l)
print("ds chain=${c} run $i", round(d["value"]), round(d["ms_per_step"],1), d["clocks"]["sm_mhz"], {k:round(v["ms_per_step"],1) for k,v in d["kernels"].items() if "gemm" in k})
PY
done
done
for i in 1 2; do
for c in off on; do
  timeout 400 python bench.py --config llama_moe --other-configs "" --rounds 0 --error-tokens 0 --no-cpu-baseline --chain $c > gpurun_out/ab_ll_${c}_$i.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/ab_ll_${c}_$i.log") if x.startswith("{")][-1]; d=json.loads(l)
print("llama chain=${c} run $i", round(d["value"]), round(d["ms_per_step"],1), d["clocks"]["sm_mhz"], {k:round(v["ms_per_step"],1) for k,v in d["kernels"].items() if "gemm" in k})
PY
done
done
