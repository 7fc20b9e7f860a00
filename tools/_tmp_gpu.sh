timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in pdl lockeys; do echo "== $v"; FHPG_LIB=$PWD/paper_1208_2428_b200/lib/ab/$v.so python tools/height_sweep.py | tail -1; done
bash tools/ab_bench.sh pdl lockeys
