set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; echo TESTS $? >> gpurun_out/r02_gpu_tests.log
timeout 300 python bench.py > gpurun_out/r02_bench_c5.log 2>&1
timeout 300 python bench.py --roots 8 --no-cpu-baseline > gpurun_out/r02_bench_c5_8roots.log 2>&1
timeout 300 python bench.py --roots 64 --steps 5 --no-cpu-baseline > gpurun_out/r02_bench_c5_64roots.log 2>&1
for c in C1 C2 C3 D2 D10; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_bench_$c.log 2>&1; done
for c in C2 D2 D10; do timeout 300 python bench.py --config $c --tf32 --no-cpu-baseline > gpurun_out/r02_bench_${c}_tf32.log 2>&1; done
timeout 600 python bench.py --config C4 --steps 5 --no-cpu-baseline > gpurun_out/r02_bench_C4.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_c5_v21.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv23 -s 3 -c 1 -o gpurun_out/r02_conv23_v21 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c23.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zhead -s 3 -c 1 -o gpurun_out/r02_zhead_v2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_zh.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_conv1_sib -s 3 -c 1 -o gpurun_out/r02_conv1_v22 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
python bench.py --config D10 --tf32 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_dnn_tc|k_mlp_tc" -c 12 -o gpurun_out/r02_tf32_d10_v5 python bench.py --config D10 --tf32 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tf.log 2>&1
echo ALLDONE
