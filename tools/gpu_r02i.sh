set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02i_gputests.log
python bench.py --config 4 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/r02i_c4.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/r02i_c4.json'));print('c4', d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks'])"
B=$GRAFT_REPO_ROOT/paper_1406_2628_b200/bin/mergebench_b200
mkdir -p /tmp/mb && cd /tmp/mb
$B gen --dist uniform --na 16777216 --nb 16777216 --seed 1 --out-a a.bin --out-b b.bin
for mem in pinned pageable; do $B merge --a a.bin --b b.bin --threads 8 --reps 5 --residency host --host-memory $mem --format csv; done
