#!/usr/bin/env python3
"""bench.py -- Merge Path on B200: the BASELINE.json headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2]
    python bench.py --impl reference ...     # the reference's CPU path

Default workload (BASELINE.json configs[1], the merge the metric is quoted
on): stable merge of two sorted int32 arrays, |A| = |B| = 2^28, keys
uniform in [0,1024) from seeds 1 (A) and 2 (B) (SURVEY.md §8d generator).
A "step" is one pass of the hot path (K1 tile partition + K2 tile merge)
over that input, resident in HBM.  Inputs (2 GiB) and output (2 GiB) are
far larger than the 126 MB L2, so no L2 flush is needed between steps.

Prints ONE JSON line (rank 0).  `value` = merged elements/s over all ranks,
device-timed with CUDA events, max over ranks; `e2e` = the same metric
through the public C ABI with host (pinned) buffers, H2D + D2H included;
`roofline` = the tile-merge kernel's algorithmic bytes / its average
CUDA-event duration vs the measured HBM peak; `cpu_baseline` = the
reference's own parallel_merge_into (oracle/_ref) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, only if the file is absent


def load_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------
CONFIGS = {
    "1": dict(kind="merge", key="u32", gen=(0, 0), na=1 << 20, nb=1 << 20, bytes_per=8,
              desc="config1: stable merge u32 |A|=|B|=2^20, seeds 1/2"),
    "2": dict(kind="merge", key="i32", gen=(1, 1), na=1 << 28, nb=1 << 28, bytes_per=8,
              desc="config2: stable merge i32 |A|=|B|=2^28, keys uniform in [0,1024), seeds 1/2"),
    "3a": dict(kind="merge", key="u64", gen=(2, 2), na=1 << 29, nb=1 << 25, bytes_per=24, vals=True,
               desc="config3a: stable merge u64 key + u32 value, |A|=2^29 |B|=2^25, uniform keys"),
    "3b": dict(kind="merge", key="u64", gen=(4, 3), na=1 << 29, nb=1 << 25, bytes_per=24, vals=True,
               desc="config3b: stable merge u64 key + u32 value, |A|=2^29 |B|=2^25, B below A"),
    "4": dict(kind="sort", key="u32", gen=(0, None), n=1 << 30, bytes_per=160,
              desc="config4: stable merge sort of 2^30 u32 keys, seed 4: 16384-key block sort + 16 merge "
                   "rounds (run as 8 fused round pairs)"),
    "5": dict(kind="merge", key="f32", gen=(5, 6), na=1 << 31, nb=1 << 31, bytes_per=8, sharded=True,
              desc="config5: stable merge f32 |A|=|B|=2^31, A~Normal(0,1), B~Exp(1), IEEE "
                   "totalOrder (one GPU: the whole merge; --gpus 8: sharded)"),
}
BARE_RUN = 16384  # mp_sort's block-sort run for bare 32-bit keys (K3w: 512 threads x 32)


def config_dict(cfg, ws):
    """The `config` object of a line -- identical for both arms (the
    reference arm's CPU thread count is in its cpu_baseline)."""
    units = cfg["n"] if cfg["kind"] == "sort" else cfg["na"] + cfg["nb"]
    alg = units * cfg["bytes_per"]
    return {"workload": cfg["desc"],
            "l2": ("inputs+output larger than L2 (no flush needed)" if alg > 4 * 126e6
                   else "fits in L2 (warm)"),
            "parallelism": f"dp{ws}" if ws > 1 else "single GPU",
            "elements_per_gpu": units}


def sort_rounds(n: int, run: int = BARE_RUN) -> int:
    """Merge rounds of mp_sort after the block sort (runs double per round)."""
    r, w = 0, run
    while w < n:
        w, r = 2 * w, r + 1
    return r


KT = {"u32": 0, "i32": 1, "f32": 2, "u64": 3, "i64": 4}
KSIZE = {"u32": 4, "i32": 4, "f32": 4, "u64": 8, "i64": 8}


def torch_dtype(torch, key):
    return {"u32": torch.uint32, "i32": torch.int32, "u64": torch.uint64,
            "i64": torch.int64, "f32": torch.float32}[key]


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while running."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake_slowdown": 0x80}
    NOTED = {"sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in {**self.BAD, **self.NOTED}.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# distributed plumbing
# --------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # smoke-testing the multi-rank path on a one-GPU box: every rank on one
    # device (MP_BENCH_DEVICE) with gloo plumbing (MP_BENCH_BACKEND=gloo)
    if "MP_BENCH_DEVICE" in os.environ:
        local = int(os.environ["MP_BENCH_DEVICE"])
    return ws, rank, local


def barrier(dist_on):
    if dist_on:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, dist_on: bool) -> float:
    if not dist_on:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def make_inputs(torch, N, cfg, dev, stream):
    """Generate the config's inputs on the device (same bytes as the oracle
    generator, tests/test_gpu_parity.py) and sort them with our own sort
    (not timed)."""
    key = cfg["key"]
    dt = torch_dtype(torch, key)
    kt = KT[key]
    s = stream.cuda_stream

    def gen(kind, seed, n):
        x = torch.empty(n, dtype=dt, device=dev)
        N.check(N.lib.mp_generate(kind, seed, 0, n, x.data_ptr(), s))
        return x

    if cfg["kind"] == "sort":
        return gen(cfg["gen"][0], 4, cfg["n"])
    a = gen(cfg["gen"][0], 1, cfg["na"])
    b = gen(cfg["gen"][1], 2, cfg["nb"])
    for x in (a, b):
        N.check(N.lib.mp_sort(kt, x.data_ptr(), None, x.numel(), None, 0, s))
    av = bv = None
    if cfg.get("vals"):
        av = torch.arange(cfg["na"], dtype=torch.int32, device=dev).view(torch.uint32)
        bv = (torch.arange(cfg["nb"], dtype=torch.int32, device=dev)
              + torch.iinfo(torch.int32).min).view(torch.uint32)
    return a, b, av, bv


def run_ours(args, cfg, ws, rank, local, dist_on):
    import torch
    from paper_1406_2628_b200 import _native as N
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    peak, peak_src = load_peak()
    key, kt = cfg["key"], KT[cfg["key"]]
    launches = 0
    with torch.cuda.stream(stream):
        if cfg["kind"] == "merge":
            a, b, av, bv = make_inputs(torch, N, cfg, dev, stream)
            na, nb = a.numel(), b.numel()
            n = na + nb
            out = torch.empty(n, dtype=a.dtype, device=dev)
            outv = torch.empty(n, dtype=torch.uint32, device=dev) if av is not None else None
            wsb = N.lib.mp_merge_workspace_bytes(kt, na, nb)
            wsp = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
            ptr = (lambda t: t.data_ptr() if t is not None else None)

            def step(evs=None):
                # mp_merge == mp_merge_plan (K1) + mp_merge_execute (K2); the
                # two-phase form lets the events isolate K2 for the roofline
                N.check(N.lib.mp_merge_plan(kt, a.data_ptr(), na, b.data_ptr(), nb,
                                            wsp.data_ptr(), stream.cuda_stream))
                if evs is not None:
                    evs[0].record(stream)
                N.check(N.lib.mp_merge_execute(kt, a.data_ptr(), ptr(av), na, b.data_ptr(),
                                               ptr(bv), nb, out.data_ptr(), ptr(outv),
                                               wsp.data_ptr(), stream.cuda_stream))
                if evs is not None:
                    evs[1].record(stream)
            launches_per_step = None  # K1 + K2 (K2 alone for a one-wave merge), measured
            units = n
        else:
            data0 = make_inputs(torch, N, cfg, dev, stream)
            n = data0.numel()
            data = torch.empty_like(data0)
            scratch_b = N.lib.mp_sort_scratch_bytes(kt, 0, n)
            scratch = torch.empty(scratch_b, dtype=torch.uint8, device=dev)

            def step(evs=None):
                # out-of-place sort: the block sort reads the unsorted keys,
                # the rounds ping-pong between `data` and the scratch
                if evs is not None:
                    evs[0].record(stream)
                N.check(N.lib.mp_sort_to(kt, data0.data_ptr(), None, data.data_ptr(), None, n,
                                         scratch.data_ptr(), scratch_b, stream.cuda_stream))
                if evs is not None:
                    evs[1].record(stream)
            launches_per_step = None  # measured on the first warm-up step
            units = n

        c_w = N.lib.mp_launch_count()
        for _ in range(args.warmup):
            step()
        stream.synchronize()
        if launches_per_step is None:  # the library's own count for one step
            launches_per_step = (N.lib.mp_launch_count() - c_w) // max(1, args.warmup)
        barrier(dist_on)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        c0 = N.lib.mp_launch_count()
        with ClockSampler(local) as clk:
            t0.record(stream)
            for i in range(args.steps):
                step(evs[i])
                launches += launches_per_step
            t1.record(stream)
            stream.synchronize()
        torch.cuda.synchronize()
        counted = N.lib.mp_launch_count() - c0
        if counted != launches:
            raise RuntimeError(f"launch count {counted} != expected {launches}")
        barrier(dist_on)
        ms = t0.elapsed_time(t1)
        kern_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in evs)
        # workloads that fit in L2 (config 1): also time each step after an
        # L2 flush (a 512 MiB write between steps; SURVEY 8d asks for warm
        # and flushed times)
        flushed = None
        step_bytes = (units * cfg["bytes_per"]) if cfg["kind"] == "merge" else units * 8
        if step_bytes <= 4 * 126e6:
            junk = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            fl = []
            for _ in range(min(args.steps, 50)):
                junk.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                stream.synchronize()
                fl.append(e0.elapsed_time(e1))
            del junk
            fms = statistics.median(fl)
            flushed = {"ms_per_step": fms, "value": units * ws / (fms / 1e3),
                       "steps": len(fl), "note": "median of single steps, each after a "
                       "512 MiB write that evicts L2 (the warm line above reuses L2)"}
    ms = max_over_ranks(ms, dist_on)
    ms_per_step = ms / args.steps
    value = units * ws * args.steps / (ms / 1e3)

    if cfg["kind"] == "merge":
        alg_bytes = n * cfg["bytes_per"]  # read A+B once, write S once
        kname = ("merge_tiles_kernel (K2); step = K1 grid-snapped split search + K2"
                 if launches_per_step > 1 else
                 "merge_tiles_kernel with in-CTA split search (one-wave merge: one launch)")
    else:
        alg_bytes = n * 8 * (1 + sort_rounds(n))
        kname = ("mp_sort: block_sort_warp + 8 x fused round pair (quad_partition + quad_refine + "
                 "quad_tile); algorithmic bytes count every round as a full pass (SURVEY 8d), the "
                 "fused pairs move half of them")
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic, traffic_src = None, "no ncu capture for this config"
    tpath = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if tpath.exists():
        # ncu DRAM bytes of the same kernel(s), stamped with the kernel
        # sources' hash: used only while the kernels are unchanged
        from paper_1406_2628_b200 import kernel_sources_sha256
        tj = json.loads(tpath.read_text())
        if tj.get("kernel_sources_sha256") == kernel_sources_sha256():
            traffic = tj.get("dram_bytes_per_launch")
            traffic_src = f"{tpath.relative_to(ROOT)} ({tj.get('source')}; kernel sources unchanged)"
        else:
            traffic_src = f"{tpath.relative_to(ROOT)} is stale (kernel sources changed since capture)"
    result = {
        "metric": "merged elements/s" if cfg["kind"] == "merge" else "merge-sort keys/s",
        "value": value,
        "unit": "elements/s" if cfg["kind"] == "merge" else "keys/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": key,
        "data": "synthetic: SplitMix64 counter generator x_i=mix64(seed+i*0x9E3779B97F4A7C15), "
                "sorted ascending before timing",
        "config": config_dict(cfg, ws),
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": kern_ms},
    }
    result["clocks"] = clk.summary()
    if flushed:
        result["l2_flushed"] = flushed
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, cfg, torch, N, dev, local, dist_on, ws)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, a if cfg["kind"] == "merge" else data0,
                                              b if cfg["kind"] == "merge" else None,
                                              out if cfg["kind"] == "merge" else None, args)
    return result


def run_e2e(args, cfg, torch, N, dev, local, dist_on, ws):
    """The same metric through the public host-buffer C ABI entry point
    (mp_merge_host / mp_sort_host): pinned host inputs in, host output back,
    all copies inside the timed region (wall clock around the synchronous
    calls)."""
    import numpy as np
    key, kt = cfg["key"], KT[cfg["key"]]
    steps = max(1, min(args.steps, args.e2e_steps))
    with torch.cuda.device(dev):
        if cfg["kind"] == "merge":
            a, b, av, bv = make_inputs(torch, N, cfg, dev, torch.cuda.current_stream())
            sample = None
            if a.numel() + b.numel() > (1 << 30):  # host RAM: 2^28-prefixes
                a, b = a[: 1 << 28].contiguous(), b[: 1 << 28].contiguous()
                sample = "2^28-element prefixes of A and B (host RAM bound)"
            ha = a.cpu().pin_memory()
            hb = b.cpu().pin_memory()
            n = a.numel() + b.numel()
            hout = torch.empty(n, dtype=a.dtype).pin_memory()
            hav = hbv = houtv = None
            if av is not None:
                hav, hbv = av.cpu().pin_memory(), bv.cpu().pin_memory()
                houtv = torch.empty(n, dtype=torch.uint32).pin_memory()
            del a, b, av, bv
            torch.cuda.synchronize()
            p = (lambda t: t.data_ptr() if t is not None else None)

            def call():
                N.check(N.lib.mp_merge_host(kt, ha.data_ptr(), p(hav), ha.numel(), hb.data_ptr(),
                                            p(hbv), hb.numel(), hout.data_ptr(), p(houtv), local))
            h2d = (ha.numel() + hb.numel()) * KSIZE[key] + (n * 4 if hav is not None else 0)
            d2h = n * KSIZE[key] + (n * 4 if hav is not None else 0)
        else:
            x = make_inputs(torch, N, cfg, dev, torch.cuda.current_stream())
            hx = x.cpu().pin_memory()
            hout = torch.empty_like(hx).pin_memory()
            n = x.numel()
            del x

            def call():
                N.check(N.lib.mp_sort_host(kt, hx.data_ptr(), None, n, hout.data_ptr(), None, local))
            h2d = d2h = n * KSIZE[key]
        for _ in range(min(2, args.warmup)):
            call()
        barrier(dist_on)
        t = time.perf_counter()
        for _ in range(steps):
            call()
        el = time.perf_counter() - t
        barrier(dist_on)
        # the same call on pageable memory (numpy arrays: what a std::vector
        # caller of the drop-in passes): staged through pinned slots
        pg = None
        if not dist_on:
            if cfg["kind"] == "merge":
                pa_, pb_ = ha.numpy().copy(), hb.numpy().copy()
                po_ = np.empty_like(hout.numpy())
                pav = hav.numpy().copy() if hav is not None else None
                pbv = hbv.numpy().copy() if hbv is not None else None
                pov = np.empty_like(houtv.numpy()) if houtv is not None else None
                q = (lambda x: x.ctypes.data if x is not None else None)

                def pcall():
                    N.check(N.lib.mp_merge_host(kt, q(pa_), q(pav), len(pa_), q(pb_), q(pbv),
                                                len(pb_), q(po_), q(pov), local))
            else:
                px_ = hx.numpy().copy()
                po_ = np.empty_like(px_)

                def pcall():
                    N.check(N.lib.mp_sort_host(kt, px_.ctypes.data, None, n, po_.ctypes.data,
                                               None, local))
            pcall()
            psteps = max(1, min(steps, 3))
            t = time.perf_counter()
            for _ in range(psteps):
                pcall()
            pel = time.perf_counter() - t
            pg = {"value": n * psteps / pel, "steps": psteps,
                  "note": "same call on pageable host arrays (staged through pinned slots)"}
    el = max_over_ranks(el, dist_on)
    unit = "elements/s" if cfg["kind"] == "merge" else "keys/s"
    del np
    return {"value": n * ws * steps / el, "unit": unit, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "api": "mp_merge_host" if cfg["kind"] == "merge" else "mp_sort_host",
            "memory": "pinned",
            **({"pageable": pg} if pg else {}),
            **({"sample": sample} if cfg["kind"] == "merge" and sample else {})}


# --------------------------------------------------------------------------
# reference (CPU) arm and cpu_baseline
# --------------------------------------------------------------------------
def ref_inputs_from_device(cfg, a, b):
    """Host copies of the same input bytes the GPU arm uses."""
    import numpy as np
    if cfg["kind"] == "sort":
        return a.cpu().numpy(), None
    ha, hb = a.cpu().numpy(), b.cpu().numpy()
    if cfg.get("vals"):
        from oracle.bindings import KV_DTYPE
        ka = np.zeros(len(ha), dtype=KV_DTYPE)
        ka["key"], ka["val"] = ha, np.arange(len(ha), dtype=np.uint32)
        kb = np.zeros(len(hb), dtype=KV_DTYPE)
        kb["key"], kb["val"] = hb, np.arange(len(hb), dtype=np.uint32) | np.uint32(1 << 31)
        return ka, kb
    return ha, hb


def host_inputs(cfg):
    """Generate the config's inputs on the host with the C restatement's
    generator (used when no GPU ran first, i.e. --impl reference)."""
    import numpy as np
    from oracle import bindings as B
    P = B.port()
    if cfg["kind"] == "sort":
        return P.generate(cfg["gen"][0], 4, 0, cfg["n"]), None
    a = P.radix_sort(P.generate(cfg["gen"][0], 1, 0, cfg["na"]))
    b = P.radix_sort(P.generate(cfg["gen"][1], 2, 0, cfg["nb"]))
    if cfg.get("vals"):
        from oracle.bindings import KV_DTYPE
        ka = np.zeros(len(a), dtype=KV_DTYPE)
        ka["key"], ka["val"] = a, np.arange(len(a), dtype=np.uint32)
        kb = np.zeros(len(b), dtype=KV_DTYPE)
        kb["key"], kb["val"] = b, np.arange(len(b), dtype=np.uint32) | np.uint32(1 << 31)
        return ka, kb
    return a, b


def time_reference(cfg, ha, hb, reps, budget_s, sample_frac=None, p=None):
    """Time the reference's own CPU path: parallel_merge_into with a warm
    thread_team(p = host cores) (parallel.hpp:151-162), or
    parallel_merge_sort(span, p) (sort.hpp:132-148).  Returns
    (elements per second, seconds per rep, p, sample description, out,
    the per-rep seconds)."""
    from oracle import bindings as B
    R = B.ref()
    p = p or B.host_cores()
    S = "kv" if cfg.get("vals") else cfg["key"]
    if cfg["kind"] == "merge":
        import numpy as np
        team = R.team(p)
        out = np.empty(len(ha) + len(hb), dtype=B.DTYPES[S])
        for _ in range(2):  # warm the team
            R.merge(S, ha, hb, team=team, out=out)
        times = []
        t_start = time.perf_counter()
        for _ in range(reps):
            t = time.perf_counter()
            R.merge(S, ha, hb, team=team, out=out)
            times.append(time.perf_counter() - t)
            if time.perf_counter() - t_start > budget_s:
                break
        team.close()
        sec = statistics.median(times)
        n = len(ha) + len(hb)
        sample = (f"full config input ({n} elements), parallel_merge_into with a warm "
                  f"thread_team({p}), median of {len(times)} reps")
        return n / sec, sec, p, sample, out, times
    # sort: a bounded prefix of the same keys (full 2^30 takes ~40 s on 8 threads)
    n = len(ha)
    m = n if sample_frac is None else max(1 << 20, int(n * sample_frac))
    d = ha[:m]
    times = []
    for _ in range(max(1, reps)):
        t = time.perf_counter()
        out, _ = R.merge_sort(S, d, p=p)
        times.append(time.perf_counter() - t)
        if sum(times) > budget_s:
            break
    sec = statistics.median(times)
    sample = (f"first {m} of the {n} config keys, parallel_merge_sort(span, p={p}) incl. its "
              f"copy/alloc, median of {len(times)} reps")
    return m / sec, sec, p, sample, out, times


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_worker(spec: str) -> int:
    """Hidden mode (--cpu-worker JSON): one fresh process times the
    reference on the inputs saved by cpu_baseline (BASELINE.md §3 / SURVEY
    H1: thread placement differs between process launches)."""
    import numpy as np
    d = json.loads(spec)
    cfg = CONFIGS[d["config"]]
    ha = np.load(d["a"], mmap_mode="r")
    hb = np.load(d["b"], mmap_mode="r") if d.get("b") else None
    ha = np.ascontiguousarray(ha)
    hb = np.ascontiguousarray(hb) if hb is not None else None
    _, _, p, _, _, times = time_reference(cfg, ha, hb, reps=d["reps"], budget_s=d["budget"],
                                          sample_frac=d.get("frac"), p=d["p"])
    print(json.dumps({"p": p, "times": times}), flush=True)
    return 0


def cpu_baseline(cfg, a, b, out_dev, args):
    """The reference's CPU path on this box's host cores:
    >= 3 separate process launches at p = host cores, one at p = 1, each
    reporting every rep; value = the median over all p = cores reps.  The
    first in-process run also verifies the GPU output against it."""
    from oracle import bindings as B
    if not B.REF_LIB.exists():
        return {"value": None, "unit": None, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    import subprocess
    import tempfile
    import numpy as np
    prefix = None
    if cfg["kind"] == "merge" and a.numel() + b.numel() > (1 << 30):
        # host-RAM bound: time (and verify) the merge of the 2^27-prefixes
        prefix = 1 << 27
        a, b = a[:prefix], b[:prefix]
    ha, hb = ref_inputs_from_device(cfg, a, b)
    frac = None if cfg["kind"] == "merge" else 1 / 16
    val, sec, p, sample, out, _ = time_reference(cfg, ha, hb, reps=3, budget_s=10,
                                                 sample_frac=frac)
    if prefix:
        sample = "2^27-element prefixes of A and B (host RAM bound); " + sample
    unit = "elements/s" if cfg["kind"] == "merge" else "keys/s"
    units = (len(ha) + len(hb)) if cfg["kind"] == "merge" else max(1 << 20, int(len(ha) * frac))
    res = {"value": val, "unit": unit, "cores": p, "kind": "reference", "sample": sample,
           "cpu_model": cpu_model(), "seconds_per_rep": sec}
    if out_dev is not None:  # verify before report (mergebench.cpp:263-265)
        if prefix:
            from paper_1406_2628_b200 import mergepath as mp
            out_dev = mp.parallel_merge(a.contiguous(), b.contiguous(), 1)
        got = out_dev.cpu().numpy()
        if got.dtype == np.float32:
            got = got.view(np.uint32)
        want = out["key"] if cfg.get("vals") else out
        res["gpu_output_bit_exact_vs_reference"] = bool(got.tobytes() == want.tobytes())
    del out
    launches = []
    with tempfile.TemporaryDirectory(prefix="mp_cpu_") as tmp:
        fa = os.path.join(tmp, "a.npy")
        np.save(fa, ha if cfg["kind"] == "merge" else ha[:units])  # the sort's sample only
        fb = None
        if hb is not None:
            fb = os.path.join(tmp, "b.npy")
            np.save(fb, hb)
        cfg_name = next(k for k, v in CONFIGS.items() if v is cfg)
        runs = [(p, 5, 10.0)] * 3 + [(1, 3, 15.0)]
        if cfg_name == "1" and p != 8:
            runs += [(8, 5, 10.0)] * 3  # config 1 is specified at p = 8
        for pp, reps, budget in runs:
            spec = json.dumps({"config": cfg_name, "a": fa, "b": fb, "p": pp, "reps": reps,
                               "budget": budget, "frac": None})
            r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--cpu-worker", spec],
                               capture_output=True, text=True, timeout=300)
            if r.returncode != 0:
                launches.append({"p": pp, "error": r.stderr[-300:]})
                continue
            d = json.loads(r.stdout.strip().splitlines()[-1])
            launches.append({"p": pp, "median_s": statistics.median(d["times"]),
                             "min_s": min(d["times"]), "reps": len(d["times"])})
    ok = [x for x in launches if "median_s" in x and x["p"] == p]
    if ok:
        med = statistics.median(x["median_s"] for x in ok)
        res.update({"value": units / med, "seconds_per_rep": med,
                    "median_s": med, "min_s": min(x["min_s"] for x in ok),
                    "sample": sample.split(", median of")[0] + f"; median over {len(ok)} "
                              "process launches x 5 reps (one more in-process run checks the "
                              "GPU output)"})
    p1 = [x for x in launches if "median_s" in x and x["p"] == 1]
    if p1 and ok:
        res["p1"] = {"value": units / p1[0]["median_s"], "median_s": p1[0]["median_s"],
                     "min_s": p1[0]["min_s"]}
        res["speedup_vs_p1"] = p1[0]["median_s"] / res["median_s"]
    p8 = [x for x in launches if "median_s" in x and x["p"] == 8 and p != 8]
    if p8:
        m8 = statistics.median(x["median_s"] for x in p8)
        res["p8"] = {"value": units / m8, "median_s": m8, "min_s": min(x["min_s"] for x in p8)}
    res["launches"] = launches
    return res


def run_reference(args, cfg, ws, rank):
    """--impl reference: the reference's own CPU implementation on this box's
    host cores, same config/metric/unit; each step = one full merge (or a
    bounded sort sample)."""
    if rank != 0:
        return None
    from oracle import bindings as B
    if not B.REF_LIB.exists():
        return {"impl": "reference", "unavailable": "oracle/_ref/libmergepath_ref.so not built"}
    ha, hb = host_inputs(cfg)
    S = "kv" if cfg.get("vals") else cfg["key"]
    R = B.ref()
    p = B.host_cores()
    times = []
    if cfg["kind"] == "merge":
        import numpy as np
        team = R.team(p)
        out = np.empty(len(ha) + len(hb), dtype=B.DTYPES[S])
        for _ in range(args.warmup):
            R.merge(S, ha, hb, team=team, out=out)
        for _ in range(args.steps):
            t = time.perf_counter()
            R.merge(S, ha, hb, team=team, out=out)
            times.append(time.perf_counter() - t)
        team.close()
        units = len(ha) + len(hb)
        sample = (f"full config input per step ({units} elements), parallel_merge_into, "
                  f"warm thread_team({p})")
    else:
        m = max(1 << 20, len(ha) // 64)
        d = ha[:m]
        for _ in range(min(args.warmup, 1)):
            R.merge_sort(S, d, p=p)
        for _ in range(args.steps):
            t = time.perf_counter()
            R.merge_sort(S, d, p=p)
            times.append(time.perf_counter() - t)
        units = m
        sample = f"first {m} config keys per step, parallel_merge_sort(span, p={p})"
    total = sum(times)
    value = units * len(times) / total
    unit = "elements/s" if cfg["kind"] == "merge" else "keys/s"
    return {
        "impl": "reference",
        "metric": "merged elements/s" if cfg["kind"] == "merge" else "merge-sort keys/s",
        "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / len(times) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg["key"], "data": "synthetic (same generator)",
        "config": config_dict(cfg, ws),
        "cpu_baseline": {"value": value, "unit": unit, "cores": p, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------------
def _spawn_ranks(args_n: int, argv) -> int:
    """--gpus N > 1 without a launcher: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1 (the driver's own
    launch line), so the requested GPU count is never silently ignored."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(args_n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "bench.py")] + list(argv)
    return subprocess.call(cmd)


def _summary(res):
    """The nested record of a secondary workload in the same run."""
    keep = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "scaling", "dtype",
            "config", "gpu_launches", "roofline", "nvlink", "clocks", "e2e", "cpu_baseline")
    return {k: res[k] for k in keep if k in res}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="only the --config workload (default: the config-2 line also "
                         "carries the sort (config 4) and, at N > 1, config 5)")
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.cpu_worker:
        return cpu_worker(args.cpu_worker)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    ws, rank, local = dist_env()
    if args.gpus < 1:
        print(json.dumps({"error": "--gpus must be >= 1"}), flush=True)
        return 2
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return _spawn_ranks(args.gpus, argv)
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr, flush=True)
        return 2
    dist_on = ws > 1
    if args.impl == "reference":
        res = run_reference(args, cfg, ws, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return 0
    if dist_on:
        import torch
        import torch.distributed as dist
        if "MP_BENCH_DEVICE" not in os.environ and torch.cuda.device_count() < ws:
            print(f"bench.py: {ws} ranks but {torch.cuda.device_count()} GPUs", file=sys.stderr)
            return 2
        torch.cuda.set_device(local)
        backend = os.environ.get("MP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    extra = not args.no_extra and args.config == "2"
    if dist_on:
        from paper_1406_2628_b200.multigpu import bench_distributed, bench_distributed_sort
        clock = (lambda: ClockSampler(local))  # noqa: E731
        if cfg["kind"] == "merge":
            res = bench_distributed(args, cfg, ws, rank, local, clock)
        else:
            res = bench_distributed_sort(args, cfg, ws, rank, local, clock)
        if extra:
            import torch
            torch.cuda.empty_cache()
            k = max(3, args.steps // 10)
            sub = argparse.Namespace(**{**vars(args), "steps": k, "warmup": 3})
            res["config5"] = _summary(bench_distributed(sub, CONFIGS["5"], ws, rank, local,
                                                        clock))
            torch.cuda.empty_cache()
            res["sort"] = _summary(bench_distributed_sort(sub, CONFIGS["4"], ws, rank, local,
                                                          clock))
    else:
        res = run_ours(args, cfg, ws, rank, local, dist_on)
        if extra:
            import torch
            torch.cuda.empty_cache()
            sub = argparse.Namespace(**{**vars(args), "config": "4",
                                        "steps": max(3, args.steps // 10)})
            res["sort"] = _summary(run_ours(sub, CONFIGS["4"], ws, rank, local, dist_on))
    if rank == 0:
        print(json.dumps(res), flush=True)
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
