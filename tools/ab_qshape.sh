# A/B of the K5e thread shape (fused two-round pass), all with MP_SORT_QUAD=1
export MP_SORT_QUAD=1
for v in base q288_31 q320_27 base q288_31 q320_27; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/qs_$v.json 2>> gpurun_out/qs_$v.err
done
for v in q288_31 q320_27; do
  MP_NATIVE_LIB=tools/variants/lib$v.so ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:quad_tile -c 1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep -E "quad_tile|duration|inst_exec|issue|registers" >> gpurun_out/qs_ncu.log
done
