# fused two-round pass: parity (quad tests) + bench + launch list
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round" > gpurun_out/qc_tests.log 2>&1; echo rc=$? >> gpurun_out/qc_tests.log
bash tools/quad_probe.sh
