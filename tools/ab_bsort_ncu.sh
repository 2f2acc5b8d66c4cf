# ncu pipe/stall breakdown of the two 16-keys-per-thread block sorts (K3t, K3w)
for k in tr merge; do
  MP_K3W=$k ncu --section ComputeWorkloadAnalysis --section WarpStateStats --section InstructionStats --section MemoryWorkloadAnalysis_Tables --clock-control none -k regex:block_sort -c 1 -f -o gpurun_out/bs_$k python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bs_$k.log 2>&1
done
