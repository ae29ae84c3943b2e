# ncu --set full of every best kernel in a bench --best-out file (run under gpurun, one GPU):
#   bash tools/profile_best.sh tools/data/best.json TAG
# then, here: python tools/ncu_summary.py TAG --traffic tools/data/best.json gpurun_out/prof_TAG_*.ncu-rep
BEST=$1; TAG=$2
for w in R G A Q L; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 \
    -o gpurun_out/prof_${TAG}_$w python tools/profile_one.py $w best $BEST --iters 8 > gpurun_out/prof_${TAG}_$w.log 2>&1
  echo "ncu $w rc $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgm_cand -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --workloads G --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-e2e-opt --tune-top 1 --best-iters 20 > /dev/null 2>&1
echo "launch list rc $?"
