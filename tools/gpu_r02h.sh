set -x
python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?"
B=paper_1406_2628_b200/bin/mergebench_b200
mkdir -p /tmp/mb && cd /tmp/mb
$GRAFT_REPO_ROOT/$B gen --n 16777216 --dist uniform --seed 1 --out a.bin && $GRAFT_REPO_ROOT/$B gen --n 16777216 --dist uniform --seed 2 --out b.bin
for mem in pinned pageable; do $GRAFT_REPO_ROOT/$B merge --a a.bin --b b.bin --threads 8 --reps 5 --residency host --host-memory $mem --format csv; done
cd $GRAFT_REPO_ROOT
python -c "import json;d=json.load(open('gpurun_out/r02h_bench.json'));print(d['value'], d['e2e']);print(d['sort']['value'], d['sort']['e2e'])"
