T=${1:-r02d}; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests/test_gpu_c5.py -x -q -rs > gpurun_out/$T/pytest_c5.log 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_c5.log
timeout 300 python tools/profile_factor.py c5p > gpurun_out/$T/factor_c5p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_front_global -s 8 -c 2 -o gpurun_out/$T/front_c5p python tools/profile_factor.py c5p > gpurun_out/$T/ncu_front.log 2>&1
timeout 1700 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/$T/bench_c5.json 2> gpurun_out/$T/bench_c5.err
