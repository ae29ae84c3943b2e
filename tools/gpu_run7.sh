set -x
python -c "from paper_2604_15272_b200 import build as B; B.build_lib()" > gpurun_out/build.log 2>&1
R=profiles/records/r01c_top20.json
for W in G A R L Q; do timeout 300 python tools/trace_one.py $W best $R > gpurun_out/trace_$W.log 2>&1; done
timeout 300 python tools/trace_one.py G "O.1.x,Wgate.1.x,Wup.1.x" '{"x":1,"i":1}' > gpurun_out/trace_G1.log 2>&1
timeout 300 python tools/trace_one.py G "O.1.x,Wgate.1.x,Wup.1.x" '{"x":1,"i":1}' '{"max_cluster":2}' > gpurun_out/trace_G1c2.log 2>&1
timeout 300 python tools/trace_one.py G "O.1.x,Wgate.1.x,Wup.1.x" '{"x":128,"i":1}' '{"max_cluster":2}' > gpurun_out/trace_G128c2.log 2>&1
timeout 300 python tools/trace_one.py R "O.1.x,W.1.x" '{"x":128,"i":1}' > gpurun_out/trace_R128.log 2>&1
tail -n 40 gpurun_out/trace_*.log
