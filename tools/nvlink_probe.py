"""NVLink pull rate between the GPUs of one box, single process.

For every ordered pair (src GPU s, dst GPU d), s != d, with peer access on:
  * "ce":  one cudaMemcpyPeerAsync-style copy (torch dst.copy_(src), copy
           engine) of SIZE MiB per transfer;
  * "sm":  mp_peer_copy on GPU d reading GPU s's buffer with SM vector loads
           (LDG.128 over NVLink -- the access pattern of the merge kernels'
           peer loader);
and "all-to-one-next": every GPU d pulls from (d+1) % N at once (SM loads),
the pattern of bench.py --gpus N's in-run probe.  CUDA events on the
launching stream; median of REPS.  With one GPU it reports the same-device
copy rates only (no NVLink), saying so.

    python tools/nvlink_probe.py [SIZE_MIB=1024] [REPS=5] > profiles/rNN/nvlink_probe.jsonl
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1406_2628_b200 import _native as N  # noqa: E402

MIB = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nbytes = MIB << 20
G = torch.cuda.device_count()
bufs = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)]
dsts = [torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)]
for g in range(G):
    bufs[g].fill_(g)


def timed(dev, fn):
    st = torch.cuda.current_stream(dev)
    ts = []
    for i in range(REPS + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(dev):
            e0.record(st)
            fn(st)
            e1.record(st)
        e1.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1) / 1e3)
    return nbytes / statistics.median(ts) / 1e9


if G == 1:
    gb = timed(0, lambda st: N.check(N.lib.mp_peer_copy(dsts[0].data_ptr(), bufs[0].data_ptr(),
                                                          nbytes, st.cuda_stream)))
    print(json.dumps({"pair": "0->0", "method": "sm", "GBps": gb,
                      "note": "one GPU visible: same-device copy, no NVLink"}))
    sys.exit(0)
for d in range(G):
    for s in range(G):
        if s == d:
            continue
        ce = timed(d, lambda st: dsts[d].copy_(bufs[s], non_blocking=True))
        sm = timed(d, lambda st: N.check(N.lib.mp_peer_copy(
            dsts[d].data_ptr(), bufs[s].data_ptr(), nbytes, st.cuda_stream)))
        print(json.dumps({"pair": f"{s}->{d}", "ce_GBps": ce, "sm_GBps": sm}), flush=True)
# all GPUs pull at once from the next one (SM loads)
for g in range(G):
    torch.cuda.synchronize(g)
evs = []
for d in range(G):
    with torch.cuda.device(d):
        st = torch.cuda.current_stream(d)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(REPS):
            N.check(N.lib.mp_peer_copy(dsts[d].data_ptr(), bufs[(d + 1) % G].data_ptr(), nbytes,
                                       st.cuda_stream))
        e1.record(st)
        evs.append((e0, e1))
rates = []
for d, (e0, e1) in enumerate(evs):
    e1.synchronize()
    rates.append(REPS * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
print(json.dumps({"pattern": "all GPUs pull from (d+1)%N at once", "method": "sm",
                  "GBps_per_gpu": rates, "min": min(rates)}))
