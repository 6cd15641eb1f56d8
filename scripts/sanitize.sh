#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py: memcheck, racecheck, synccheck,
# initcheck on every mode; logs in gpurun_out/sanitizer/ (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
out=gpurun_out/sanitizer
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool mode [env]
    local tool=$1 mode=$2 envs=$3
    env $envs timeout 900 $CS --tool $tool --error-exitcode 17 --print-limit 20 \
        python scripts/sanitize_run.py $mode > $out/${tool}_${mode}.log 2>&1
    echo "$tool $mode ($envs): rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|done' $out/${tool}_${mode}.log | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck initcheck; do
    run $tool default
    run $tool staged MRF_K5=staged
    run $tool voxel MRF_K6=voxel
    run $tool compact MRF_COMPACT=1
    run $tool long
    run $tool kfavg
    run $tool sparse
    run $tool mf
done 2>&1 | tee $out/summary.txt
