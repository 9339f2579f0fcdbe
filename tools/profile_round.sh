#!/bin/bash
# Round profiling (run on the GPU box via gpurun): the launch list of one bench invocation and
# `ncu --set full` captures of every hot kernel.  Outputs land in gpurun_out/; summarise them into
# profiles/ with tools/ncu_summary.py (runs without a GPU).   usage: bash tools/profile_round.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --error-tokens 0 --rounds 0 --other-configs "" \
  > gpurun_out/prof_bench_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"router|permute|grouped_gemm|combine" -c 5 \
  -o gpurun_out/layer_$tag -f python tools/micro.py layer > gpurun_out/prof_layer_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"router|permute|grouped_gemm|combine" -c 5 \
  -o gpurun_out/llama_layer_$tag -f python tools/micro.py layer_llama > gpurun_out/prof_llama_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"quantize_kernel|dequant_kernel" -c 2 \
  -o gpurun_out/quant_$tag -f python tools/micro.py layer > gpurun_out/prof_quant_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"merge" -c 1 \
  -o gpurun_out/merge_$tag -f python tools/micro.py merge_model > gpurun_out/prof_merge_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gram_kernel|gram_reduce|eig_kernel|kmeans_kernel" -c 4 \
  -o gpurun_out/cluster_$tag -f python tools/micro.py features > gpurun_out/prof_cluster_$tag.log 2>&1
ls -la gpurun_out
