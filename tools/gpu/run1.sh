# GPU session 1: parity tests (headline teacher-forced, fp32 mode), GPU suite, short bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests/test_parity_fp32_gpu.py -x -q -s > gpurun_out/t_fp32.log 2>&1; echo fp32 rc $?
timeout 1500 python -m pytest tests/test_headline_parity_gpu.py -x -q -s > gpurun_out/t_headline.log 2>&1; echo headline rc $?
timeout 1200 python -m pytest tests -m gpu -q -k "not headline and not fp32" > gpurun_out/t_gpu.log 2>&1; echo gpu rc $?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench rc $?
tail -3 gpurun_out/t_fp32.log gpurun_out/t_headline.log gpurun_out/t_gpu.log
tail -c 1500 gpurun_out/bench1.log
