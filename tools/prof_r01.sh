set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_pipe.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tma_gemm --launch-skip 20 --launch-count 1 -o gpurun_out/ncu_dw_l1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_bwd --launch-skip 7 --launch-count 1 -o gpurun_out/ncu_spmm_bwd_l2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_fwd --launch-skip 9 --launch-count 1 -o gpurun_out/ncu_spmm_fwd_l1 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
