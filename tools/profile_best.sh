# ncu --set full of every best kernel (and its runners-up) in a bench --best-out file
# (run under gpurun, one GPU):
#   bash tools/profile_best.sh gpurun_out/best.json TAG
# then, here: python tools/ncu_summary.py TAG --traffic gpurun_out/best.json gpurun_out/prof_TAG_*.ncu-rep
BEST=$1; TAG=$2
for w in R G A Q L; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 \
    -o gpurun_out/prof_${TAG}_$w python tools/profile_one.py $w best $BEST --iters 8 > gpurun_out/prof_${TAG}_$w.log 2>&1
  echo "ncu $w rc $?"
  for k in 0 1 2; do
    timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof_${TAG}_${w}_ru$k \
      python tools/profile_one.py $w best $BEST --iters 8 --runner-up $k > gpurun_out/prof_${TAG}_${w}_ru$k.log 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --workloads G --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-e2e-opt --tune-top 1 --best-iters 20 > /dev/null 2>&1
echo "launch list rc $?"
