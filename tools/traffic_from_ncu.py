"""Write profiles/traffic_config<C>.json from an ncu launch list with DRAM
metrics (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv ... python bench.py
--config C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra`).

The file is stamped with the SHA-256 of the kernel sources
(paper_1406_2628_b200.kernel_sources_sha256()); bench.py reports
`roofline.traffic` from it only while the sources are unchanged, and null
(stale) otherwise.

    python tools/traffic_from_ncu.py LAUNCHES.csv CONFIG KERNEL_REGEX [STEP_KERNELS]

KERNEL_REGEX picks the dominant kernel for a merge (per-launch bytes of its
last launch = the timed steps'); for the sort (config 4) give "step" and the
whole last sort (the launches of one step, STEP_KERNELS of them, from the
end of the list) is summed."""
from __future__ import annotations

import collections
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def launches(path):
    lines = Path(path).read_text().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = [r for r in csv.reader(lines[start:]) if len(r) > 10]
    h = rows[0]
    ix = {x: i for i, x in enumerate(h)}
    by_id = collections.OrderedDict()
    for r in rows[1:]:
        if r[0] == "ID":
            continue
        d = by_id.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return list(by_id.values())


def main():
    from paper_1406_2628_b200 import kernel_sources_sha256
    path, config, pat = sys.argv[1], sys.argv[2], sys.argv[3]
    L = launches(path)
    rd, wr, us = "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"
    if pat == "step":
        k = int(sys.argv[4])
        step = L[-k:]
        per = collections.OrderedDict()
        for x in step:
            n = re.sub(r"\(.*", "", x["name"]).replace("void ", "")
            d = per.setdefault(n, {"launches": 0, "dram_bytes_read": 0.0,
                                   "dram_bytes_write": 0.0, "duration_us": 0.0})
            d["launches"] += 1
            d["dram_bytes_read"] += x.get(rd, 0.0)
            d["dram_bytes_write"] += x.get(wr, 0.0)
            d["duration_us"] += x.get(us, 0.0) / 1e3
        r = sum(d["dram_bytes_read"] for d in per.values())
        w = sum(d["dram_bytes_write"] for d in per.values())
        out = {"kernel": "one mp_sort step (all launches)", "config": config,
               "dram_bytes_read": r, "dram_bytes_write": w, "dram_bytes_per_launch": r + w,
               "duration_us_sum_of_kernels": sum(d["duration_us"] for d in per.values()),
               "per_kernel": per}
    else:
        hits = [x for x in L if re.search(pat, x["name"])]
        x = hits[-1]
        out = {"kernel": re.sub(r"\(.*", "", x["name"]).replace("void ", ""), "config": config,
               "dram_bytes_read": x.get(rd), "dram_bytes_write": x.get(wr),
               "dram_bytes_per_launch": x.get(rd, 0) + x.get(wr, 0),
               "duration_us": x.get(us, 0) / 1e3}
    out["source"] = str(Path(path).relative_to(ROOT)) if Path(path).is_absolute() else path
    out["kernel_sources_sha256"] = kernel_sources_sha256()
    dst = ROOT / "profiles" / f"traffic_config{config}.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(dst, out["dram_bytes_per_launch"])


if __name__ == "__main__":
    main()
