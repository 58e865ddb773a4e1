# GPU session 11: branch-group model tests + Inception-v3 launch list + bench line
set -x
timeout 1500 python -m pytest tests/test_branchy_gpu.py -q -s > gpurun_out/t_branchy.log 2>&1; echo branchy rc $?
timeout 600 python tools/model_launches.py inception-v3 2 > gpurun_out/inc_plain.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_inception.csv python tools/model_launches.py inception-v3 2 > gpurun_out/ncu_inc.log 2>&1; echo list rc $?
timeout 900 python bench.py --steps 10 --warmup 3 --no-fp32 > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo bench rc $?
tail -3 gpurun_out/t_branchy.log; cat gpurun_out/inc_plain.log | tail -2
