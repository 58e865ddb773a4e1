# GPU session 30: AlexNet (BASELINE config 2) headline line + launch list
set -x
timeout 600 python bench.py --model alexnet --steps 20 --warmup 5 --quick > gpurun_out/bench_alex.json 2> gpurun_out/bench_alex.err; echo bench rc $?
timeout 600 python tools/model_launches.py alexnet 4 > gpurun_out/alex_plain.log 2>&1; echo plain rc $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_alexnet.csv python tools/model_launches.py alexnet 2 > gpurun_out/ncu_alex.log 2>&1; echo list rc $?
cut -c1-300 gpurun_out/bench_alex.json; tail -1 gpurun_out/alex_plain.log
