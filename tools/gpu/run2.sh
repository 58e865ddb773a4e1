# GPU session 2: parity tests, HEAD launch list with DRAM/tensor counters, ncu full captures
set -x
timeout 1200 python -m pytest tests/test_parity_fp32_gpu.py -q -s > gpurun_out/t_fp32.log 2>&1; echo fp32 rc $?
timeout 1500 python -m pytest tests/test_headline_parity_gpu.py -q -s > gpurun_out/t_headline.log 2>&1; echo headline rc $?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
timeout 300 python tools/step_launches.py 2 > gpurun_out/plain_steps.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_r02.csv python tools/step_launches.py 2 > gpurun_out/ncu_list.log 2>&1; echo list rc $?
for pat in "conv_slab_fwd_kernel<3, 4, 1, true>" "conv_slab_wgrad_pair_kernel" "conv_first_fwd_kernel" "maxpool_bwd_disjoint" "conv_row64_kernel" "gemm_sm100_kernel" "conv_slab_fwd_kernel<3, 4, 1, false>"; do
  tag=$(echo "$pat" | tr -c 'a-z0-9_' '_' | cut -c1-40)
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$pat" -c 1 -o gpurun_out/prof_$tag python tools/step_launches.py 1 > gpurun_out/ncu_$tag.log 2>&1; echo cap $tag rc $?
done
tail -n 3 gpurun_out/t_fp32.log gpurun_out/t_headline.log
