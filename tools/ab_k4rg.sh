# A/B: K4r guess window (default 128)
for v in ${K4RG_VARIANTS:-base k4rg64 k4rg256}; do
  if [ $v = base ]; then L=""; else L="tools/variants/lib$v.so"; fi
  MP_NATIVE_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:quad_refine -c 8 --csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep quad_refine | awk -F'","' -v v=$v '{gsub(/"/,"",$NF); s+=$NF} END {print v, s/1000, "us total for 8 launches"}' >> gpurun_out/k4rg.log
  MP_NATIVE_LIB=$L python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/k4rg_$v.json 2>/dev/null
done
