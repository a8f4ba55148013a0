# round-2 pass 5: full GPU suite, wgrad micro-bench, device timelines, consumer-fused BERT rows, default bench
mkdir -p gpurun_out
export OPTFUSE_PARITY_OUT=gpurun_out/r02_c1_parity.json
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --durations=20 --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -8
timeout 600 python tools/wgrad_bench.py > gpurun_out/wgrad_bench.json 2> gpurun_out/wgrad_bench.err; echo wgrad_bench=$?; cat gpurun_out/wgrad_bench.json | head -60
for c in c2 c3 c5; do timeout 600 python tools/device_timeline.py $c > gpurun_out/device_timeline_$c.json 2> gpurun_out/device_timeline_$c.err; echo timeline_$c=$?; head -12 gpurun_out/device_timeline_$c.json; done
timeout 2400 python bench.py --extras c5m --standalone 0 --in-situ 0 --extras-out gpurun_out/bench_extras_c5m.json > gpurun_out/bench_c5m.log 2> gpurun_out/bench_c5m.err; echo bench_c5m=$?; tail -3 gpurun_out/bench_c5m.err
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?; tail -c 2200 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
