# round-2 session-3 pass C: split-K cluster wgrad kernel -- parity, micro-bench, ncu, consumer-fused BERT rows
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest -q -m gpu tests/test_wgrad_fused_gpu.py tests/test_consumer_fusion_gpu.py > gpurun_out/pytest_c.log 2>&1; echo pytest_c=$?; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_c.log | tail -8
timeout 600 python tools/wgrad_bench.py > gpurun_out/wgrad_bench.json 2> gpurun_out/wgrad_bench.err; echo wgrad_bench=$?
python -c "
import json; d=json.load(open('gpurun_out/wgrad_bench.json'))
for r in d['rows']: print(r['layer'], 'fused', r['fused_us'], 'unfused', r['unfused_us'], 'cublas', r['cublas_gemm_us'], 'TF', r['fused_tflops'], r['cublas_tflops'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad -c 3 -o gpurun_out/prof_wgrad -f python tools/wgrad_bench.py > gpurun_out/ncu_wgrad.log 2>&1; echo ncu_wgrad=$?
for r in gpurun_out/prof_wgrad.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  rm -f "$r"
done
if [ -n "${C5M}" ]; then
timeout 2400 python bench.py --extras c5m --standalone 0 --in-situ 0 --extras-out gpurun_out/bench_extras_c5m.json > gpurun_out/bench_c5m.log 2> gpurun_out/bench_c5m.err; echo bench_c5m=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_extras_c5m.json'))
for s,r in d['c5m']['schedules'].items(): print('%-60s %8.3f %s'%(s,r['ms_per_step'],r.get('speedup_vs_ours_unfused','')))"
fi
# residency of the C3 / C5 backward kernels (room for a co-resident update CTA?)
for cfg in c3 c5; do
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_static,launch__shared_mem_per_block_dynamic,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_warps,launch__occupancy_limit_blocks,launch__waves_per_multiprocessor \
  --clock-control none --nvtx --nvtx-include "iter" -c 5000 --csv --log-file gpurun_out/residency_$cfg.csv python tools/iter_dram.py $cfg baseline > gpurun_out/residency_$cfg.log 2>&1; echo residency_$cfg=$?
done
timeout 900 python -m pytest -q -m gpu tests/test_kernels_gpu.py -k capped > gpurun_out/pytest_capped.log 2>&1; echo pytest_capped=$?; tail -1 gpurun_out/pytest_capped.log
for c in ${CONTENTION:-c3 c5 c4}; do timeout 1500 python tools/bf_contention.py $c 3 > gpurun_out/bf_narrow_$c.json 2> gpurun_out/bf_narrow_$c.err; echo narrow_$c=$?; python -c "
import json,sys; d=json.load(open('gpurun_out/bf_narrow_$c.json'))
for k,v in list(d.values())[0].items(): print(k, v['median_ms'], v['vs_baseline'])" ; done
