# GPU session 3: parity (triples), headline SGD diagnostics, bench, ncu captures of the dominant kernels
set -x
timeout 1500 python -m pytest tests/test_parity_fp32_gpu.py -q -s > gpurun_out/t_fp32.log 2>&1; echo fp32 rc $?
timeout 900 python -m pytest tests/test_headline_parity_gpu.py -q -s -k "sgd or split" > gpurun_out/t_headline_sgd.log 2>&1; echo headline rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo bench rc $?
python tools/step_launches.py 1 > gpurun_out/plain_steps.log 2>&1 && echo plain ok
for spec in "conv_slab_fwd_kernel<3, 4, 1, 1>:0" "conv_slab_fwd_kernel<3, 4, 1, 0>:0" "conv_slab_fwd_kernel<3, 4, 2, 1>:1" "conv_slab_wgrad_pair_kernel:6" "conv_slab_wgrad_kernel:0"; do
  pat="${spec%:*}"; skip="${spec##*:}"
  tag=$(echo "$pat" | tr -c 'a-z0-9_' '_' | cut -c1-40)
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$pat" -s $skip -c 1 -o gpurun_out/prof_$tag python tools/step_launches.py 1 > gpurun_out/ncu_$tag.log 2>&1; echo cap $tag rc $?
done
