#!/bin/bash
# Every BASELINE.json workload shape through bench.py (1 GPU, device-timed, no e2e/cpu legs):
#   bash tools/config_sweep.sh > gpurun_out/configs.jsonl
# long512k / long1m at the BASELINE B x H = 96 need more workspace than HBM holds at once: they run
# in groups of slices (--groups) with seeded inputs drawn on the device (--device-inputs: 51 GB of
# inputs at long1m); the 12- and 6-slice runs of round 1 are kept for comparison.
set -u
for c in ar ar_tokens lra_nc lra_c lra_tokens wiki wiki_tokens long64k long128k long256k; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
done
timeout 300 python bench.py --config long512k --bh 12 --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
timeout 300 python bench.py --config long1m --bh 6 --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
timeout 900 python bench.py --config long512k --groups 4 --device-inputs --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
timeout 1200 python bench.py --config long1m --groups 16 --device-inputs --steps 3 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1
