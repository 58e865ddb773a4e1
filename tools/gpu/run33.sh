set -x
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_step_gpu.py -q -x > gpurun_out/t_33.log 2>&1; echo tests rc $?
timeout 600 python tools/model_launches.py alexnet 4 > gpurun_out/alex_plain33.log 2>&1; echo plain rc $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet33.csv python tools/model_launches.py alexnet 2 > gpurun_out/ncu_alex33.log 2>&1; echo list rc $?
timeout 600 python bench.py --model alexnet --steps 30 --warmup 5 --quick > gpurun_out/bench_alex33.json 2>/dev/null; echo bench rc $?
tail -2 gpurun_out/t_33.log; tail -1 gpurun_out/alex_plain33.log; cut -c1-200 gpurun_out/bench_alex33.json
