set -x
python -c "from paper_2604_15272_b200 import build as B; B.build_lib()" > gpurun_out/build.log 2>&1
for W in G R A Q L; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof5_$W python tools/profile_one.py $W best profiles/records/r01b_top20.json --iters 8 > gpurun_out/ncu5_$W.log 2>&1; echo "ncu $W rc $?"
done
# R column split (TMA f32) for comparison
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof5_Rcol python tools/profile_one.py R "O.1.x,W.1.x" '{"x":128,"i":1}' --iters 8 > gpurun_out/ncu5_Rcol.log 2>&1; echo "ncu Rcol rc $?"
