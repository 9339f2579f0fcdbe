#!/bin/bash
# compute-sanitizer over every libflux entry point on tiny shapes (race detection).
# Run on the GPU box via gpurun; logs land in gpurun_out/, summarise into profiles/.
#   usage: bash tools/sanitize.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_driver.py > gpurun_out/san_plain_$tag.log 2>&1
echo "plain rc=$?" >> gpurun_out/san_plain_$tag.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_driver.py > gpurun_out/san_${tool}_$tag.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_${tool}_$tag.log
done
tail -n 3 gpurun_out/san_*_$tag.log
