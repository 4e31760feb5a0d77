#!/usr/bin/env python
"""Benchmark of the hot path; prints ONE JSON line on rank 0.

Main line: least-model fixpoint of configuration C4 (10M atoms, 50M rules, ~150M
nonzeros; BASELINE.json configs[3], the configuration the roofline target is quoted on)
with the full fused θ-pass kernel (Algorithm 1), v0 = facts.  A step = one whole
fixpoint (init + all θ-passes until no change + model extraction) through the C ABI,
inputs resident in HBM.  value = nnz · iters / step time, summed over ranks.

Also measured (extra keys): the frontier variant on C4, the batched stable-model search
on C5 (guesses/s), the end-to-end call with host buffers (e2e), the per-launch roofline
of the dominant kernel and the CPU oracle baseline (cpu_baseline).

--impl reference times the CPU oracle (oracle/, as it stands) on the same workload and
metric: each step is a bounded sample (one Jacobi T_P pass over all of C4's rules).

Multi-GPU (torchrun, N > 1): "replicas only" -- every rank solves its own copy of the
workload (the least-model fixpoint has no partition without a per-pass exchange; see
DESIGN.md), timing is the max over ranks, value the sum of units over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

KERNEL_REV = "lead16-octets-d2-pipe"   # bump when the dominant kernel's traffic changes
METRIC = ("least-model fixpoint time & nnz·iter/s (HBM GB/s vs peak); "
          "stable-model guesses/s")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled with NVML every ~1 ms DURING the timed
    region (a background thread between start() and stop())."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.001)

    def start(self):
        if self.nv:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()

    def stop(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.t.join(timeout=2)
        s = self.samples
        return {"sm_mhz": float(np.median(s)) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s),
                "source": "NVML every ~1 ms during the timed region"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import lpgen
    import oracle
    oracle.build()
    P = lpgen.config(args.workload)
    nnz = int(P.nnz) + int((np.diff(P.body_ptr) == 0).sum())
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, it, _, _ = oracle.lm_jacobi(P, max_iters=1)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    v = nnz * 1 / t
    sample = f"one Jacobi T_P pass over all {P.n_rules} rules of {args.workload} per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "nnz*iter/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": args.workload, "variant": "oracle O-LM Jacobi (oracle/lp_oracle.c)"},
        "cpu_baseline": {"value": v, "unit": "nnz*iter/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "nnz*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--stable-workload", default="C5")
    ap.add_argument("--no-extras", action="store_true", help="main line only (for ncu)")
    ap.add_argument("--cpu-sample-reps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import lpgen
    from paper_2009_10247_b200 import lp

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1 or os.environ.get("BENCH_FORCE_DIST"):   # (FORCE: exercise the N>1 code on one GPU)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.Stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def flush_l2():
        with torch.cuda.stream(stream):
            flush.fill_(rank + 1)

    # ---- load the workload (not timed: lp_load is the one-time upload) --------------
    t0 = time.perf_counter()
    P = lpgen.config(args.workload)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    prog = lp.Program(P, device=local)
    torch.cuda.synchronize()
    t_load = time.perf_counter() - t0
    info = prog.info
    n = P.n_atoms
    Wm = lp.bits_words(n)
    launches_per_call = 1      # lp_least_model = one cooperative launch (prologue..extraction)

    model = torch.zeros(Wm, dtype=torch.int64, device="cuda")
    iters_d = torch.zeros(1, dtype=torch.int32, device="cuda")
    stats_d = torch.zeros(6, dtype=torch.int64, device="cuda")

    def timed_least_model(frontier, steps, warmup):
        tot, ker, byts, mhz = [], [], [], []
        for i in range(warmup + steps):
            flush_l2()
            e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e0.record(stream)
            lp.lp_least_model(prog, None, model, frontier=frontier, stream=stream, device_ptrs=True,
                              iters_out=iters_d, ev_begin=k0, ev_end=k1, stats=stats_d)
            e1.record(stream)
            stream.synchronize()
            if i >= warmup:
                tot.append(e0.elapsed_time(e1))
                ker.append(k0.elapsed_time(k1))
                sd = stats_d.tolist()
                byts.append(int(sd[0]))
                if sd[5] > 0:
                    mhz.append(1e3 * sd[4] / sd[5])
        dev_clock.extend(mhz)
        if tot:
            trial_stats.update(mean_ms=float(np.mean(tot)), median_ms=float(np.median(tot)),
                               min_ms=float(np.min(tot)), stdev_ms=float(np.std(tot)), trials=len(tot))
        return (float(np.mean(tot)) if tot else 0.0, float(np.mean(ker)) if ker else 0.0,
                int(iters_d.item()), float(np.mean(byts)) if byts else 0.0,
                [int(x) for x in stats_d.tolist()])

    # ---- main line: full θ-pass fixpoint ---------------------------------------------
    dev_clock = []
    trial_stats = {}
    clocks = ClockSampler(local)
    timed_least_model(False, 0, args.warmup)            # warm-up
    barrier()
    clocks.start()
    dev_clock.clear()
    ms, kms, iters, alg_bytes, st = timed_least_model(False, args.steps, 0)
    main_trials = dict(trial_stats)
    barrier()
    clk = clocks.stop()
    # the SM clock each timed launch actually ran at (%clock64 / %globaltimer in-kernel)
    clk["nvml_sm_mhz"] = clk.get("sm_mhz")
    if dev_clock:
        clk["sm_mhz"] = float(np.median(dev_clock))
        clk["sm_mhz_min"] = float(np.min(dev_clock))
        clk["source"] = ("sm_mhz: device %clock64/%globaltimer over each timed launch (median); "
                         "reasons: NVML every ~1 ms during the timed region")
    ms_max = allmax(ms)
    kms_max = allmax(kms)
    nnz = int(info["nnz"])
    value = ws * nnz * iters / (ms_max / 1e3)

    hbm_peak, peak_src = _peaks()
    # algorithmic bytes of the launch, counted by the kernel itself (lp_run.stats_out):
    # the planes each pass streamed + 4 B per body entry / head the verification loaded +
    # 12 B per derived atom
    alg_bytes = allmax(alg_bytes)
    achieved = alg_bytes / (kms_max / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.workload)
        if tr and tr["passes_per_launch"] == iters and tr.get("kernel_rev") == KERNEL_REV:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram bytes per launch)",
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                "kernel": "lm_full_kernel<false> (persistent: all passes of the fixpoint in one launch)",
                "passes_per_launch": iters, "lead_passes": st[1], "rows_verified": st[2],
                "lead_pass_bytes": int(info["lead_pass_bytes"]),
                "stream_pass_bytes": int(info["stream_pass_bytes"]), "kernel_ms": kms_max}

    out = {
        "metric": METRIC, "value": value, "unit": "nnz*iter/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.workload, "n_atoms": n, "n_rules": int(info["n_rules"]),
                   "nnz": nnz, "iters": iters, "variant": "full fused θ-pass (Algorithm 1)",
                   "v0": "facts only", "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "truth_mode": "summary-in-smem" if info["truth_mode"] else "exact-in-smem",
                   "grid": [int(info["grid_blocks"]), int(info["block_threads"])]},
        "fixpoint_ms": ms_max, "kernel_ms": kms_max, "trials": main_trials,
        "gpu_launches": launches_per_call * args.steps,
        "roofline": roofline, "clocks": clk,
        "load": {"generate_s": t_gen, "lp_load_s": t_load, "device_bytes": int(info["device_bytes"])},
    }

    # ---- e2e: the C-ABI call with host (pinned) buffers -------------------------------
    v0_host = torch.zeros(Wm, dtype=torch.int64).pin_memory()
    model_host = torch.zeros(Wm, dtype=torch.int64).pin_memory()
    facts = P.head[np.diff(P.body_ptr) == 0]
    v0_np = lp.pack_mask(np.isin(np.arange(n), facts))
    v0_host.numpy().view(np.uint64)[:] = v0_np[:Wm]
    e2e_t = []
    for i in range(args.warmup + args.steps):
        flush_l2()
        stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        it = lp.lp_least_model(prog, v0_host, model_host, stream=stream)
        e1.record(stream)
        e1.synchronize()
        if i >= args.warmup:
            e2e_t.append(e0.elapsed_time(e1))
        assert it == iters
    e2e_ms = allmax(float(np.mean(e2e_t)))
    out["e2e"] = {"value": ws * nnz * iters / (e2e_ms / 1e3), "unit": "nnz*iter/s",
                  "h2d_bytes_per_step": Wm * 8, "d2h_bytes_per_step": Wm * 8 + 12,
                  "ms_per_step": e2e_ms, "api": "lp_least_model (host pointers, synchronous)"}

    if not args.no_extras and dist:
        # ---- strong-scaling extra: ONE C4 least model sharded by head ranges over the
        # ranks, one all-gather + OR per pass (shard.py) -------------------
        from paper_2009_10247_b200.shard import ShardedLeastModel
        sharded = ShardedLeastModel(P)             # setup: head range, sub-program upload
        sh_t = []
        for i in range(1 + min(args.steps, 5)):
            flush_l2()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m_sh, it_sh, _ = sharded.run(popcounts=False)
            e1.record()
            torch.cuda.synchronize()
            if i >= 1:
                sh_t.append(e0.elapsed_time(e1))
        assert it_sh == iters
        sh_ms = allmax(float(np.mean(sh_t)))
        out["sharded"] = {"ms_per_step": sh_ms, "value": nnz * iters / (sh_ms / 1e3),
                          "unit": "nnz*iter/s", "iters": it_sh, "ranks": ws,
                          "what": "one program, head ranges per rank, all-gather + OR per pass"}
        del sharded

    if not args.no_extras:
        # ---- the 8-bit key plane (LP_LOAD_KEY8) on the same workload: fewer bytes per
        # pass, which then stay L2-resident across passes ----------
        prog8 = lp.Program(P, device=local, frontier=False, key8=True)
        k8 = []
        for i in range(args.warmup + args.steps):
            flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lp.lp_least_model(prog8, None, model, stream=stream, device_ptrs=True, iters_out=iters_d,
                              stats=stats_d)
            e1.record(stream)
            stream.synchronize()
            if i >= args.warmup:
                k8.append(e0.elapsed_time(e1))
        assert int(iters_d.item()) == iters
        k8ms = allmax(float(np.mean(k8)))
        out["key8"] = {"ms_per_step": k8ms, "value": ws * nnz * iters / (k8ms / 1e3), "unit": "nnz*iter/s",
                       "algorithmic_bytes_per_launch": int(stats_d[0].item()),
                       "lead_pass_bytes": int(prog8.info["lead_pass_bytes"]),
                       "note": "8-bit key codes: the per-pass plane fits L2, so this variant is "
                               "L2/latency-bound, not HBM-bound (ncu: profiles/r01_ncu_full_c4_key8.md)"}
        prog8.close()

        # ---- frontier variant on the same workload --------------------------------------
        fms, fkms, fit, _, _ = timed_least_model(True, args.steps, args.warmup)
        assert fit == iters
        out["frontier"] = {"ms_per_step": allmax(fms), "kernel_ms": allmax(fkms), "iters": fit,
                           "speedup_vs_full": ms_max / allmax(fms)}
        # ---- stable models ---------------------------------------------------------------
        # guess-sharded under torchrun: rank r solves its 64-aligned slice
        # of the 2^f guesses (lp_run.guess_offset), no exchange until the final gather
        from paper_2009_10247_b200.shard import guess_slices, stable_models_sharded
        S = lpgen.config(args.stable_workload)
        sprog = lp.Program(S, device=local)
        G_all = 1 << sprog.info["n_free_negated"]
        goff, G = guess_slices(G_all, ws)[rank]
        W = max((G + 63) // 64, 1)
        acc = torch.zeros(W, dtype=torch.int64, device="cuda")
        nacc = torch.zeros(1, dtype=torch.int64, device="cuda")
        passes = torch.zeros(1, dtype=torch.int32, device="cuda")
        st_t, st_k = [], []
        for i in range(args.warmup + args.steps):
            flush_l2()
            e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e0.record(stream)
            if G > 0:
                lp.lp_stable_models(sprog, None, G, acc, stream=stream, device_ptrs=True,
                                    n_accepted_out=nacc, passes_out=passes, ev_begin=k0,
                                    ev_end=k1, guess_offset=goff)
            else:
                k0.record(stream)
                k1.record(stream)
            e1.record(stream)
            stream.synchronize()
            if i >= args.warmup:
                st_t.append(e0.elapsed_time(e1))
                st_k.append(k0.elapsed_time(k1))
        sms = allmax(float(np.mean(st_t)))
        stable = {"workload": args.stable_workload, "guesses": G_all,
                  "guesses_per_s": G_all / (sms / 1e3), "ms_per_step": sms,
                  "kernel_ms": allmax(float(np.mean(st_k))), "passes": int(allmax(int(passes.item()))),
                  "accepted": int(nacc.item()), "n_negated": sprog.info["n_negated"],
                  "l2": "flushed between steps", "launches_per_call": 1,
                  "sharding": f"guesses over {ws} rank(s), slice time max over ranks"}
        if dist:
            ids, ps = stable_models_sharded(sprog, sprog.info["n_free_negated"])
            stable["accepted"], stable["passes"] = int(ids.size), ps
        out["stable"] = stable
        sprog.close()

    # ---- CPU baseline: the oracle as it stands, rank 0, N = 1 only ----------------------
    if rank == 0 and ws == 1:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        reps, it_cpu = 0, 0
        while reps < args.cpu_sample_reps and (reps == 0 or time.perf_counter() - t0 < 10.0):
            _, it1, _, conv = oracle.lm_jacobi(P)      # the whole fixpoint, as it stands
            assert conv and it1 == iters
            it_cpu += it1
            reps += 1
        dt = time.perf_counter() - t0
        cpu_model = ""
        try:
            with open("/proc/cpuinfo") as f:
                cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
        except OSError:
            pass
        out["cpu_baseline"] = {"value": nnz * it_cpu / dt, "unit": "nnz*iter/s", "cores": 1,
                               "kind": "oracle", "cpu": cpu_model, "host_cores": os.cpu_count(),
                               "sample": f"{reps} whole fixpoint(s) of O-LM Jacobi (oracle/lp_oracle.c, "
                                         f"{it_cpu} T_P passes over all of {args.workload}, {dt:.1f} s, "
                                         f"single thread)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
