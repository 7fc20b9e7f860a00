# memory-pipeline calibration + stream-only timing builds
./tools/membw > gpurun_out/membw_r02b.json 2>&1; cat gpurun_out/membw_r02b.json
rm -f gpurun_out/ab.txt; bash tools/ab_bench.sh base so1 so2 so3 so5 so6
