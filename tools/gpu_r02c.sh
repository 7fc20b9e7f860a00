timeout 900 python -m pytest tests/test_planes_gpu.py tests/test_parity_gpu.py -q -x > gpurun_out/pytest_r02c.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_r02c.log
rm -f gpurun_out/ab.txt; bash tools/ab_bench.sh ring pair15 pair16
