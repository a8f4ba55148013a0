# Whole-iteration DRAM traffic per schedule (ncu, one iteration each; see tools/iter_dram.py).
#   CONFIGS="c3 c4 c5" bash tools/iter_dram.sh      -> gpurun_out/iter_dram_<cfg>_<sched>.csv
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c2 c3 c4 c5}; do
  for sched in ${SCHEDS:-baseline bf1 bf2 ff}; do
    timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --cache-control none --clock-control none --nvtx --nvtx-include "iter" -c 5000 --csv \
      --log-file gpurun_out/iter_dram_${cfg}_${sched}.csv python tools/iter_dram.py $cfg $sched \
      > gpurun_out/iter_dram_${cfg}_${sched}.log 2>&1
    echo "iter_dram $cfg $sched rc=$?"
  done
done
python tools/summarize_iter_dram.py gpurun_out > gpurun_out/iter_dram_summary.md 2>&1; echo summary=$?
cat gpurun_out/iter_dram_summary.md | head -60
