# one gpurun call: gpu tests, a bench line, optional ncu (NCU=1) of the three gather kernels
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputest.log
python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${CONFIGS:-}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
done
if [ "${NCU:-0}" = 1 ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${NCU_K:-topk_attn_fwd|bwd_query|bwd_key}" -c ${NCU_C:-3} -o /tmp/src python tools/prof_step.py --config long64k --steps 1 > gpurun_out/ncu.log 2>&1
for k in ${NCU_K_LIST:-topk_attn_fwd bwd_query bwd_key}; do
  ncu -i /tmp/src.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>>gpurun_out/ncu.log
done
ncu -i /tmp/src.ncu-rep --page raw --csv > gpurun_out/raw_src.csv 2>>gpurun_out/ncu.log
fi
echo done
