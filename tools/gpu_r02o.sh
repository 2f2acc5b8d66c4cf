# fused passes for 64-bit keys: parity (forced at every size) and rates
set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "fused_round_sorts and (u64 or i64)" 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -1
python tools/sort_types_probe.py
MP_SORT_QUAD=0 python tools/sort_types_probe.py
