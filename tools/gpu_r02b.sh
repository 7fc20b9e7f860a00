bash tools/ab_bench.sh base dyn dynps200 dynps1000 dynts256 basets256
timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 -k "multi_gpu or observables_gpu or checkpoint" > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu_r02b.log
