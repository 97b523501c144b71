# Round-end evidence in one gpurun call (1 GPU): gpu tests, the default bench line, the ncu launch
# list of one long64k step (times + DRAM bytes per launch), an ncu --set full capture of the
# dominant kernels (summary + DRAM traffic per launch), every BASELINE shape through bench.py.
set -x
TAG=${TAG:-r02}
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py --config long64k --steps 1 > gpurun_out/ncu_launch.log 2>&1
python tools/ncu_step.py gpurun_out/launches_$TAG.csv --json gpurun_out/ncu_step_dram.json --workload long64k \
  > gpurun_out/ncu_step_${TAG}_summary.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"topk_attn_fwd|bwd_query|bwd_key|csr_count" -c 4 -o /tmp/full_$TAG \
  python tools/prof_step.py --config long64k --steps 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/full_$TAG.ncu-rep --traffic gpurun_out/ncu_traffic.json \
  > gpurun_out/ncu_full_${TAG}_summary.txt 2>&1
if [ "${SWEEP:-1}" = 1 ]; then bash tools/config_sweep.sh > gpurun_out/configs_$TAG.jsonl 2>/dev/null; fi
echo done
if [ "${SEQ:-1}" = 1 ]; then timeout 1200 python tools/seqshard_report.py > gpurun_out/seqshard_$TAG.json 2>gpurun_out/seqshard.err; fi
echo done-all
