timeout 600 ./tests/cpp/test_host_api gpu | tail -3
timeout 900 ./oracle/_ref/dropin/dropin_check check data/fhp3.fhptab > gpurun_out/dropin_r02h.txt 2>&1; echo dropin=$?; cat gpurun_out/dropin_r02h.txt
timeout 900 ./oracle/_ref/dropin/dropin_check e2e data/fhp3.fhptab 20 > gpurun_out/dropin_e2e_r02h.txt 2>&1; echo e2e=$?; cat gpurun_out/dropin_e2e_r02h.txt
timeout 600 python tools/dump_cadence.py 1000 100 32 > gpurun_out/dump_cadence_r02h.json 2>&1; echo cadence=$?; cat gpurun_out/dump_cadence_r02h.json
