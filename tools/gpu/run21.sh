# GPU session 21: the driver's default bench invocation (N=1, all comparators, CPU baseline) timed
set -x
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo bench rc $? elapsed $(( $(date +%s) - t0 ))
t0=$(date +%s); timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref21.json 2> gpurun_out/ref21.err; echo ref rc $? elapsed $(( $(date +%s) - t0 ))
cut -c1-400 gpurun_out/ref21.json
