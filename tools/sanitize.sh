#!/bin/bash
# compute-sanitizer over the whole path: memcheck, racecheck, synccheck and initcheck on
# the tiny config and two AR slices (f32 and bf16 value rows), plus the hub-key "tokens" input (long
# CSR segments) and the code-distance selection.  Summaries -> gpurun_out/sanitizer/ (copied to profiles/).
set -u
out=${1:-gpurun_out/sanitizer}
mkdir -p "$out"
run() {   # tool, label, args...
    local tool=$1 label=$2
    shift 2
    timeout 1200 compute-sanitizer --tool "$tool" --error-exitcode 99 --print-limit 20 \
        python tools/sanitize_step.py "$@" > "$out/${tool}_${label}.log" 2>&1
    echo "$tool $label rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|done' "$out/${tool}_${label}.log" | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck initcheck; do
    run $tool tiny --config tiny
    run $tool ar2 --config ar --bh 2
    run $tool ar2_bf16 --config ar --bh 2 --vdtype 1
done
run memcheck ar_tokens2 --config ar_tokens --bh 2
run racecheck ar_tokens2 --config ar_tokens --bh 2
run memcheck lra_tokens1 --config lra_tokens --bh 1
run racecheck tiny_select --config tiny --select 1
run memcheck tiny_select --config tiny --select 1
