mkdir -p gpurun_out
for pr in 0 1; do echo "== PAIR=$pr" >> gpurun_out/aux_ab.log; VEGS_FWD_PAIR=$pr timeout 600 python scripts/aux_step_time.py 5 >> gpurun_out/aux_ab.log 2>&1; done
VEGS_FWD_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "aux" >> gpurun_out/aux_ab.log 2>&1
