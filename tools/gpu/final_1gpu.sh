# Final single-GPU evidence at HEAD: full GPU suite, smoke, default bench line, reference arm,
# VGG-16 launch list (+ traffic json), ncu captures of the dominant conv kernel and an FC GEMM
set -x
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo tests rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc $?
timeout 1500 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo bench rc $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref_n1.json 2> gpurun_out/final_ref_n1.err; echo ref rc $?
timeout 600 python tools/step_launches.py 2 > gpurun_out/final_plain.log 2>&1; echo plain rc $?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches_vgg16.csv python tools/step_launches.py 2 > gpurun_out/final_ncu_list.log 2>&1; echo list rc $?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:conv_slab_fwd_kernel<.int.3, .int.4, .int.1, .bool.1>" -s 2 -c 1 -o gpurun_out/final_prof_conv_fwd_pair python tools/step_launches.py 1 > gpurun_out/final_ncu_conv.log 2>&1; echo cap rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_sm100_kernel -s 0 -c 1 -o gpurun_out/final_prof_gemm_fc1 python tools/step_launches.py 1 > gpurun_out/final_ncu_gemm.log 2>&1; echo cap rc $?
tail -3 gpurun_out/final_tests.log; tail -2 gpurun_out/final_smoke.log; cut -c1-200 gpurun_out/final_bench_n1.json; cut -c1-200 gpurun_out/final_ref_n1.json
