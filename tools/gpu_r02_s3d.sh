# pass D: wgrad probe (token sweep, ncu source-level stalls), eager launch list of the headline
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in "3072 768" "768 768"; do timeout 300 python tools/wgrad_probe.py sweep $s; done > gpurun_out/wgrad_sweep.jsonl 2> gpurun_out/wgrad_sweep.err; echo sweep=$?; cat gpurun_out/wgrad_sweep.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wgrad -s 2 -c 1 -o gpurun_out/prof_wgrad1 -f python tools/wgrad_probe.py one 3072 768 4096 > gpurun_out/ncu_wgrad1.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_wgrad1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_wgrad1.sass.csv 2>/dev/null; echo src=$?
ncu -i gpurun_out/prof_wgrad1.ncu-rep --page details --csv > gpurun_out/prof_wgrad1.details.csv 2>/dev/null
ncu -i gpurun_out/prof_wgrad1.ncu-rep --page raw --csv > gpurun_out/prof_wgrad1.raw.csv 2>/dev/null
rm -f gpurun_out/prof_wgrad1.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed" -c 3000 --csv \
  --log-file gpurun_out/launches_eager.csv python bench.py --headline-only --graphs 0 --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench_eager.log 2>&1; echo ncu_list=$?
ls -la gpurun_out
