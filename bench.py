#!/usr/bin/env python
"""Benchmark of the hot path; prints ONE JSON line on rank 0.

Main line: least-model fixpoint of configuration C4 (10M atoms, 50M rules, ~150M
nonzeros; BASELINE.json configs[3], the configuration the roofline target is quoted on)
with the full fused θ-pass kernel (Algorithm 1), v0 = facts.  A step = one whole
fixpoint (init + all θ-passes until no change + model extraction) through the C ABI,
inputs resident in HBM.  value = nnz · iters / step time.

Also measured (extra keys): the frontier variant on C4, the batched stable-model search
on C5 (guesses/s), the end-to-end call with host buffers (e2e), the per-launch roofline
of the dominant kernel and the CPU oracle baseline (cpu_baseline).

--impl reference times the CPU oracle (oracle/, as it stands) on the same workload and
metric: each step is one whole O-STAGE fixpoint of C4 on one pinned host core.

Multi-GPU (torchrun, N > 1): ONE C4 least model sharded by head ranges over the ranks
(shard.py): per pass a θ-pass of each rank's rules, an NCCL all-gather of the
owned words + status word and the device combine kernel (lp_shard_combine); "scaling":
"strong" (the same program for every N), time = max over ranks.  The stable-model search
on C5 is guess-sharded (no exchange until the final mask gather) in the "stable" key.
BENCH_FORCE_DIST=1 runs that path with one rank on one GPU.
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

KERNEL_REV = "armed-lead"   # bump when the dominant kernel's traffic changes
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


def _pinned_stage_timed(P, trials, v0=None):
    """O-STAGE's fixpoint phase (oracle.lm_stage_timed), this thread pinned to core 0
    (taskset -c 0 equivalent; BASELINE.md's CPU-baseline plan), affinity restored after."""
    import oracle
    old = os.sched_getaffinity(0)
    try:
        os.sched_setaffinity(0, {min(old)})
        return oracle.lm_stage_timed(P, v0=v0, trials=trials), min(old)
    finally:
        os.sched_setaffinity(0, old)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            return next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        return ""


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (O-STAGE forward chaining, the plan of
    BASELINE.md), single thread pinned to one core; each step = one whole fixpoint of the
    workload (occurrence lists built once beforehand, like lp_load on our side)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import lpgen
    import oracle
    oracle.build()
    P = lpgen.config(args.workload)
    nnz = int(P.nnz) + int((np.diff(P.body_ptr) == 0).sum())
    (_, _, iters, secs), core = _pinned_stage_timed(P, args.warmup + args.steps)
    times = secs[args.warmup:]
    t = float(np.mean(times))
    v = nnz * iters / t
    sample = (f"{args.steps} whole O-STAGE fixpoints of {args.workload} ({iters} T_P passes "
              f"equivalent each; occurrence lists built once, untimed), core {core}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "nnz*iter/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": args.workload, "iters": iters,
                   "variant": "oracle O-STAGE forward chaining (oracle/lp_oracle.c)"},
        "cpu_baseline": {"value": v, "unit": "nnz*iter/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": _cpu_model(), "host_cores": os.cpu_count(),
                         "median_ms": float(np.median(times)) * 1e3},
        "e2e": {"value": v, "unit": "nnz*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def _ncu_traffic(key, iters):
    """dram read+write bytes of one launch from a committed ncu capture
    (profiles/ncu_traffic.json), when its pass count and kernel revision match."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(key)
        if tr and tr["passes_per_launch"] == iters and tr.get("kernel_rev") == KERNEL_REV:
            return tr["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        pass
    return None


def _model_bytes_per_pass(info, n):
    """SURVEY.md §8(d)'s algorithmic bytes of one T_P pass over a CSR program:
    B_pass = 4·nnz + 4·(R+1) + 4·(H+1) + 2·ceil((n+1)/8) (column ids, rule delimiters,
    head grouping, truth vector read + write)."""
    return (4 * int(info["nnz"]) + 4 * (int(info["n_rules"]) + 1) + 4 * (int(info["n_heads"]) + 1)
            + 2 * ((n + 1 + 7) // 8))


def _model_bytes_per_pass_stable(info, n, W):
    """SURVEY.md §8(d)'s batched form: B_pass = 4·nnz + 4·(R+1) + 4·(H+1) + 2·(n+1+k)·W·8
    (the program, then the bit-sliced truth matrix read and written, W guess words per row)."""
    return (4 * int(info["nnz"]) + 4 * (int(info["n_rules"]) + 1) + 4 * (int(info["n_heads"]) + 1)
            + 2 * (n + 1 + int(info["n_negated"])) * W * 8)


def sprog_info_compact(stable):
    return int(stable.get("compact_atoms", 0)) > 0


def _l2_peak():
    """Measured L2 read bandwidth (tools/l2bw.cu, profiles/l2_peak.json): the denominator of
    the L2-resident stable pass's roofline."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_peak.json")) as f:
            d = json.load(f)
        return float(d["gbs"]), d.get("source", "profiles/l2_peak.json")
    except Exception:  # noqa: BLE001
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--stable-workload", default="C5")
    ap.add_argument("--no-extras", action="store_true", help="main line only (for ncu)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--cpu-trials", type=int, default=3)
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
    # L2 flush before every timed call: a 1 GiB write (8x the L2).  Its ~0.15 ms on the device
    # also covers the host's launch path (ctypes marshalling + lp_least_model), which is
    # issued while the fill runs: with a 256 MiB fill (~37 us) a slow host left the device
    # idle between the step's start event and the kernel (0.134 vs 0.088 ms on one box)
    flush = torch.empty(1024 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

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
    status_d = torch.zeros(1, dtype=torch.int32, device="cuda")

    def timed_least_model(pr, steps, warmup, frontier=False, v0=None, schedule="auto", out=None):
        """steps timed calls (device pointers, L2 flushed before each); every call's
        kernel-written status word must be 0 (fixpoint reached, nothing dropped)."""
        tot, ker, byts, mhz = [], [], [], []
        out = model if out is None else out
        for i in range(warmup + steps):
            flush_l2()
            e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e0.record(stream)
            lp.lp_least_model(pr, v0, out, frontier=frontier, stream=stream, device_ptrs=True,
                              iters_out=iters_d, ev_begin=k0, ev_end=k1, stats=stats_d,
                              schedule=schedule, status_out=status_d)
            e1.record(stream)
            stream.synchronize()
            assert int(status_d.item()) == 0, f"device status {int(status_d.item())}"
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
    timed_least_model(prog, 0, args.warmup)            # warm-up
    barrier()
    clocks.start()
    dev_clock.clear()
    ms, kms, iters, kern_bytes, st = timed_least_model(prog, args.steps, 0)
    main_trials = dict(trial_stats)
    barrier()
    clk = clocks.stop()
    main_model = model.cpu().numpy().view(np.uint64).copy()
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
    # Roofline of the dominant kernel (lm_full_kernel<false>, one launch = the fixpoint):
    #   achieved = SURVEY §8(d)'s algorithmic bytes (B_pass x passes) / kernel time, as the
    #   contract defines it.  Armed LEAD passes read only the records of the rows whose
    #   lead atom is true (not every CSR entry), so this exceeds the HBM peak: frac > 1
    #   means the work skipped,
    #   not a bandwidth.  Beside it: the bytes the kernel itself counted and the ncu DRAM
    #   bytes of one launch, each as a fraction of the peak.
    b_pass = _model_bytes_per_pass(info, n)
    model_bytes = b_pass * iters
    achieved = model_bytes / (kms_max / 1e3) / 1e9
    kern_bytes = allmax(kern_bytes)
    traffic = _ncu_traffic(args.workload, iters)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "binding": "latency: grid barriers and dependent L2 round trips per pass (armed "
                           "LEAD passes verify a few thousand rows per pass from their records)",
                "model": "SURVEY §8(d) B_pass = 4 nnz + 4 (R+1) + 4 (H+1) + 2 ceil((n+1)/8), "
                         "x passes per launch",
                "model_bytes_per_pass": b_pass, "model_bytes_per_launch": model_bytes,
                "kernel_bytes_per_launch": kern_bytes,
                "kernel_gbs": kern_bytes / (kms_max / 1e3) / 1e9,
                "kernel_frac": kern_bytes / (kms_max / 1e3) / 1e9 / hbm_peak,
                "traffic_gbs": None if traffic is None else traffic / (kms_max / 1e3) / 1e9,
                "traffic_frac": None if traffic is None else traffic / (kms_max / 1e3) / 1e9 / hbm_peak,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full: dram read+write bytes "
                                  "of one launch)",
                "peak_source": peak_src,
                "kernel": "lm_full_kernel<false> (persistent: all passes of the fixpoint in one launch)",
                "passes_per_launch": iters, "lead_passes": st[1], "rows_verified": st[2],
                "full_key_plane_bytes": int(info["lead_pass_bytes"]),
                "stream_pass_bytes": int(info["stream_pass_bytes"]), "kernel_ms": kms_max}

    out = {
        "metric": METRIC, "value": value, "unit": "nnz*iter/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.workload, "n_atoms": n, "n_rules": int(info["n_rules"]),
                   "nnz": nnz, "iters": iters, "variant": "full fused θ-pass (Algorithm 1)",
                   "v0": "facts only", "l2": "flushed between steps (1 GiB write)",
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
    # the host-buffer model equals the device-pointer main line's, word for word
    assert (model_host.numpy().view(np.uint64) == main_model).all()
    e2e_ms = allmax(float(np.mean(e2e_t)))
    out["e2e"] = {"value": ws * nnz * iters / (e2e_ms / 1e3), "unit": "nnz*iter/s",
                  "h2d_bytes_per_step": Wm * 8, "d2h_bytes_per_step": Wm * 8 + 12,
                  "ms_per_step": e2e_ms, "api": "lp_least_model (host pointers, synchronous)",
                  "model_check": "equal to the device-pointer main line's model"}

    if dist:
        # ---- N > 1 main line: ONE C4 least model sharded by head ranges over the ranks
        # (strong scaling): per pass one θ-pass per rank (owned words +
        # status word), one NCCL all-gather of the payloads, one combine kernel on the
        # device (OR, changed flag); the host reads pass k's flag after queuing pass k+1 ---
        from paper_2009_10247_b200.shard import ShardedLeastModel
        sharded = ShardedLeastModel(P)             # setup: head range, sub-program upload
        sh_t = []
        for i in range(args.warmup + args.steps):
            flush_l2()
            stream.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m_sh, it_sh, _ = sharded.run(popcounts=False)
            e1.record()
            torch.cuda.synchronize()
            if i >= args.warmup:
                sh_t.append(e0.elapsed_time(e1))
        assert it_sh == iters and (m_sh == main_model).all()
        sh_ms = allmax(float(np.mean(sh_t)))
        out["single_gpu"] = {"ms_per_step": ms_max, "kernel_ms": kms_max, "value": nnz * iters / (ms_max / 1e3),
                             "what": "the one-GPU fused fixpoint on each rank (replica)"}
        out.update(value=nnz * iters / (sh_ms / 1e3), ms_per_step=sh_ms, scaling="strong",
                   gpu_launches=2 * (iters + 1) * args.steps)
        out["config"]["parallelism"] = f"head-range shards x{ws} (one program)"
        out["config"]["variant"] = ("head-range-sharded T_P passes: per pass one θ-pass per rank, NCCL "
                                    "all-gather of owned words + status, device combine (lp_shard_combine)")
        out["sharded"] = {"ms_per_step": sh_ms, "iters": it_sh, "ranks": ws,
                          "words_per_rank": sharded.stride - 1, "lag": "host reads pass k's flag after queuing k+1"}
        # e2e: host v0 in, host model out, through the sharded public API
        v0w = lp.pack_mask(np.isin(np.arange(n), P.head[np.diff(P.body_ptr) == 0]))
        v0_pinned = torch.from_numpy(v0w.view(np.int64)).pin_memory().numpy().view(np.uint64)
        e2e_s = []
        for i in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            m_e, it_e, _ = sharded.run(v0_words=v0_pinned, popcounts=False)
            e2e_s.append(time.perf_counter() - t0)
        assert it_e == iters and (m_e == main_model).all()
        e2e_sh = allmax(float(np.mean(e2e_s[args.warmup:])) * 1e3)
        out["e2e"] = {"value": nnz * iters / (e2e_sh / 1e3), "unit": "nnz*iter/s",
                      "h2d_bytes_per_step": Wm * 8, "d2h_bytes_per_step": Wm * 8,
                      "ms_per_step": e2e_sh, "api": "shard.ShardedLeastModel.run(v0_words=pinned host words) -> host words"}
        del sharded

    if not args.no_extras:
        # ---- the regime that streams M_P: STREAM passes only (every body position, every
        # pass -- Algorithm 1's u = θ(M v) over all rows), same workload -----
        sms_, skms, sit, sbytes, sst = timed_least_model(prog, args.steps, args.warmup, schedule="stream")
        assert sit == iters and (model.cpu().numpy().view(np.uint64) == main_model).all()
        out["stream"] = {
            "ms_per_step": allmax(sms_), "kernel_ms": allmax(skms), "iters": sit,
            "value": ws * nnz * iters / (allmax(sms_) / 1e3), "unit": "nnz*iter/s",
            "roofline": {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak,
                         "kernel_bytes_per_launch": sbytes,
                         "achieved": sbytes / (allmax(skms) / 1e3) / 1e9,
                         "frac": sbytes / (allmax(skms) / 1e3) / 1e9 / hbm_peak,
                         "traffic": _ncu_traffic(args.workload + "_stream", iters),
                         "model_achieved": model_bytes / (allmax(skms) / 1e3) / 1e9,
                         "model_frac": model_bytes / (allmax(skms) / 1e3) / 1e9 / hbm_peak,
                         "note": "kernel bytes = every body plane streamed each pass (int32 ids, "
                                 "position-major) + verification; §8(d)'s model adds CSR row "
                                 "pointers and head grouping this layout does not need"}}
        # ---- v0 = facts ∪ 1 % random atoms (seeded): atoms outside D2 light the coarse key
        # buckets, so LEAD passes stream the whole key plane (HBM) -----------------------
        rng = np.random.default_rng(20251020)
        extra = rng.choice(n, size=n // 100, replace=False)
        v0r = torch.from_numpy(lp.pack_mask(np.isin(np.arange(n), np.union1d(facts, extra))).view(np.int64)).cuda()
        rmodel = torch.zeros_like(model)
        rms, rkms, rit, rbytes, rst = timed_least_model(prog, args.steps, args.warmup, v0=v0r, out=rmodel)
        rb = {"ms_per_step": allmax(rms), "kernel_ms": allmax(rkms), "iters": rit,
              "value": ws * nnz * rit / (allmax(rms) / 1e3), "unit": "nnz*iter/s",
              "lead_passes": rst[1], "rows_verified": rst[2],
              "roofline": {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak,
                           "kernel_bytes_per_launch": rbytes,
                           "achieved": rbytes / (allmax(rkms) / 1e3) / 1e9,
                           "frac": rbytes / (allmax(rkms) / 1e3) / 1e9 / hbm_peak,
                           "model_frac": b_pass * rit / (allmax(rkms) / 1e3) / 1e9 / hbm_peak},
              "v0": "facts ∪ 1% uniform random atoms (numpy seed 20251020)"}
        out["random_v0"] = rb
        del v0r, rmodel
        # ---- the same workload without armed LEAD passes (LP_NO_ARMED, read by lp_load):
        # the LEAD passes stream the live runs of the 16-bit key plane -------------------
        os.environ["LP_NO_ARMED"] = "1"
        try:
            prog8 = lp.Program(P, device=local, frontier=False)
        finally:
            del os.environ["LP_NO_ARMED"]
        assert prog8.info["armed_list_cap"] == 0
        k8ms, k8k, k8it, k8b, _ = timed_least_model(prog8, args.steps, args.warmup)
        assert k8it == iters and (model.cpu().numpy().view(np.uint64) == main_model).all()
        out["unarmed"] = {"ms_per_step": allmax(k8ms), "kernel_ms": allmax(k8k),
                          "value": ws * nnz * iters / (allmax(k8ms) / 1e3), "unit": "nnz*iter/s",
                          "kernel_bytes_per_launch": k8b,
                          "lead_pass_bytes": int(prog8.info["lead_pass_bytes"]),
                          "note": "LP_NO_ARMED: LEAD passes stream the live runs of the 16-bit key "
                                  "plane (the round-2 path before armed passes)"}
        prog8.close()

        # ---- frontier variant on the same workload --------------------------------------
        fms, fkms, fit, _, _ = timed_least_model(prog, args.steps, args.warmup, frontier=True)
        assert fit == iters and (model.cpu().numpy().view(np.uint64) == main_model).all()
        out["frontier"] = {"ms_per_step": allmax(fms), "kernel_ms": allmax(fkms), "iters": fit,
                           "speedup_vs_full": ms_max / allmax(fms)}
        # ---- the other least-model configurations (latency-bound: time only) -----------
        cfgs = {}
        for cname in ("C1", "C2", "C3"):
            Q = lpgen.config(cname)
            qp = lp.Program(Q, device=local)
            qm = torch.zeros(lp.bits_words(Q.n_atoms), dtype=torch.int64, device="cuda")
            steps_c = args.steps if cname != "C3" else max(3, args.steps // 3)
            a_ms, a_k, a_it, _, _ = timed_least_model(qp, steps_c, args.warmup, out=qm)
            f_ms, f_k, f_it, _, _ = timed_least_model(qp, steps_c, args.warmup, frontier=True, out=qm)
            assert a_it == f_it
            cfgs[cname] = {"iters": a_it, "full_ms": allmax(a_ms), "full_kernel_ms": allmax(a_k),
                           "frontier_ms": allmax(f_ms), "frontier_kernel_ms": allmax(f_k),
                           "us_per_pass_full": 1e3 * allmax(a_k) / a_it,
                           "nnz": int(qp.info["nnz"]),
                           "kernel": ("lm_small_kernel (one CTA, rows in shared memory, semi-naive row "
                                      "lists; full and frontier calls)" if qp.info["small_rows"] > 0 else
                                      "lm_cluster_kernel / one-cluster frontier" if qp.info["cluster_ctas"] > 0
                                      else "lm_full_kernel / lm_frontier_kernel (persistent grid)")}
            qp.close()
        out["configs"] = cfgs
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
                                    ev_end=k1, guess_offset=goff, status_out=status_d)
            else:
                k0.record(stream)
                k1.record(stream)
            e1.record(stream)
            stream.synchronize()
            assert G == 0 or int(status_d.item()) == 0
            if i >= args.warmup:
                st_t.append(e0.elapsed_time(e1))
                st_k.append(k0.elapsed_time(k1))
        sms = allmax(float(np.mean(st_t)))
        stable = {"workload": args.stable_workload, "guesses": G_all,
                  "guesses_per_s": G_all / (sms / 1e3), "ms_per_step": sms,
                  "kernel_ms": allmax(float(np.mean(st_k))), "passes": int(allmax(int(passes.item()))),
                  "accepted": int(nacc.item()), "n_negated": sprog.info["n_negated"],
                  "l2": "flushed between steps", "launches_per_call": 1,
                  "sharding": f"guesses over {ws} rank(s), slice time max over ranks",
                  "kernel": ("st_compact_kernel (live sub-program over A* in shared memory, a CTA "
                             "per guess word; DESIGN.md 'Compact stable kernel')"
                             if sprog.info["stable_compact_atoms"] > 0 else
                             "st_fixpoint_kernel (batched persistent grid)"),
                  "compact_atoms": sprog.info["stable_compact_atoms"],
                  "compact_rows": sprog.info["stable_compact_rows"]}
        # roofline (SURVEY §8(d) batched form): C5's program and truth matrix (~112 MB)
        # stay in the 126 MB L2 across the passes, so the bound is L2, against the measured
        # L2 read bandwidth; ncu DRAM bytes of one call beside it
        Wall = max((G_all + 63) // 64, 1)
        sb = _model_bytes_per_pass_stable(sprog.info, S.n_atoms, Wall)
        spasses = int(stable["passes"])
        l2_gbs, l2_src = _l2_peak()
        ach = sb * spasses / (stable["kernel_ms"] / 1e3) / 1e9
        stable["roofline"] = {"bound": "l2", "unit": "GB/s", "model_bytes_per_pass": sb,
                              "passes_per_launch": spasses, "achieved": ach, "peak": l2_gbs,
                              "frac": (ach / l2_gbs) if l2_gbs else None, "peak_source": l2_src,
                              "traffic": _ncu_traffic("C5_stable_compact" if sprog.info["stable_compact_atoms"] > 0
                                                      else "C5_stable", spasses),
                              "binding": ("latency: dependent shared-memory loads and two block barriers "
                                          "per pass inside one CTA per guess word (the model's bytes are "
                                          "never moved: rows outside A* cannot fire, DESIGN.md R25)"
                                          if sprog.info["stable_compact_atoms"] > 0 else
                                          "latency: grid barriers and dependent L2 round trips per pass "
                                          "(armed passes touch only the candidate rows' guess words)")}
        if dist:
            ids, ps = stable_models_sharded(sprog, sprog.info["n_free_negated"])
            stable["accepted"], stable["passes"] = int(ids.size), ps
        out["stable"] = stable
        sprog.close()
        if not dist and sprog_info_compact(stable):
            # A/B: the batched persistent-grid kernel on the same call (LP_NO_COMPACT_STABLE
            # is read by lp_load)
            os.environ["LP_NO_COMPACT_STABLE"] = "1"
            bprog = lp.Program(S, device=local)
            del os.environ["LP_NO_COMPACT_STABLE"]
            bt, bk = [], []
            for i in range(args.warmup + args.steps):
                flush_l2()
                e0, e1, k0, k1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e0.record(stream)
                lp.lp_stable_models(bprog, None, G, acc, stream=stream, device_ptrs=True,
                                    n_accepted_out=nacc, passes_out=passes, ev_begin=k0,
                                    ev_end=k1, guess_offset=goff, status_out=status_d)
                e1.record(stream)
                stream.synchronize()
                assert int(status_d.item()) == 0
                if i >= args.warmup:
                    bt.append(e0.elapsed_time(e1))
                    bk.append(k0.elapsed_time(k1))
            assert int(nacc.item()) == stable["accepted"] and int(passes.item()) == stable["passes"]
            sb_ach = sb * spasses / (float(np.mean(bk)) / 1e3) / 1e9
            out["stable_batched"] = {
                "ms_per_step": float(np.mean(bt)), "kernel_ms": float(np.mean(bk)),
                "guesses_per_s": G_all / (float(np.mean(bt)) / 1e3),
                "kernel": "st_fixpoint_kernel (batched persistent grid, armed passes; LP_NO_COMPACT_STABLE)",
                "roofline": {"bound": "l2", "unit": "GB/s", "achieved": sb_ach, "peak": l2_gbs,
                             "frac": (sb_ach / l2_gbs) if l2_gbs else None,
                             "traffic": _ncu_traffic("C5_stable", spasses)}}
            bprog.close()
        # ---- the same recipe with 16 negated atoms: 65,536 guesses = 2,048 half-words of 32
        # columns, 14 per CTA of the compact kernel (its throughput past the single wave the
        # k = 12 workload fills; sampled columns oracle-checked in tests/test_gpu_parity.py) --
        if not dist:
            S16 = lpgen.gen_c5(seed=1, n=100_000, R=500_000, k=16)
            p16 = lp.Program(S16, device=local)
            G16 = 1 << p16.info["n_free_negated"]
            acc16 = torch.zeros((G16 + 63) // 64, dtype=torch.int64, device="cuda")
            t16 = []
            for i in range(args.warmup + args.steps):
                flush_l2()
                k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                lp.lp_stable_models(p16, None, G16, acc16, stream=stream, device_ptrs=True,
                                    n_accepted_out=nacc, passes_out=passes, ev_begin=k0, ev_end=k1,
                                    status_out=status_d)
                stream.synchronize()
                assert int(status_d.item()) == 0
                if i >= args.warmup:
                    t16.append(k0.elapsed_time(k1))
            out["stable_k16"] = {"workload": "C5 recipe, k = 16 (lpgen.gen_c5(seed=1, k=16))", "guesses": G16,
                                 "kernel_ms": float(np.mean(t16)),
                                 "guesses_per_s": G16 / (float(np.mean(t16)) / 1e3),
                                 "passes": int(passes.item()), "accepted": int(nacc.item()),
                                 "compact_atoms": p16.info["stable_compact_atoms"],
                                 "kernel": "st_compact_kernel" if p16.info["stable_compact_atoms"] > 0
                                           else "st_fixpoint_kernel"}
            p16.close()
        # ---- guess-space reduction (lp_stable_search, reading R23): C5's
        # recipe with k = 32 negated atoms -- 2^32 guesses, enumeration refused (LP_E_CAP);
        # 128 sampled columns per round + local search, all rounds in one launch ----------
        S32 = lpgen.gen_c5(seed=3, n=100_000, R=500_000, k=32)
        sp32 = lp.Program(S32, device=local)
        h, kk = 128, sp32.info["n_negated"]
        gs = torch.zeros((kk, 2), dtype=torch.int64, device="cuda")
        acc2 = torch.zeros(2, dtype=torch.int64, device="cuda")
        na2 = torch.zeros(1, dtype=torch.int64, device="cuda")
        rd2 = torch.zeros(1, dtype=torch.int32, device="cuda")
        ps2 = torch.zeros(1, dtype=torch.int32, device="cuda")
        ss_t = []
        for i in range(args.warmup + args.steps):
            flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lp.lp_stable_search(sp32, h, 5, 40, gs, acc2, stream=stream, device_ptrs=True, n_accepted_out=na2,
                                rounds_out=rd2, passes_out=ps2, status_out=status_d)
            e1.record(stream)
            stream.synchronize()
            assert int(status_d.item()) == 0
            if i >= args.warmup:
                ss_t.append(e0.elapsed_time(e1))
        out["stable_search"] = {"workload": "C5 recipe, k = 32 (lpgen.gen_c5(seed=3, k=32))",
                                "columns_per_round": h, "seed": 5, "rounds": int(rd2.item()),
                                "passes": int(ps2.item()), "accepted": int(na2.item()),
                                "ms_per_search": allmax(float(np.mean(ss_t))), "launches_per_call": 1,
                                "enumeration": "2^32 guesses: lp_stable_models refuses (LP_E_CAP)"}
        sp32.close()

    # ---- CPU baseline (BASELINE.md plan): O-STAGE, fixpoint only, one pinned core, median
    # of 3 trials; rank 0 at N = 1 only.  Its model also checks the GPU main line. -------
    if rank == 0 and ws == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        (om, _, oit, secs), core = _pinned_stage_timed(P, args.cpu_trials)
        wall = time.perf_counter() - t0
        assert oit == iters and (oracle.pack_bits(om) == main_model).all(), "GPU model != oracle"
        med = float(np.median(secs))
        out["cpu_baseline"] = {"value": nnz * iters / med, "unit": "nnz*iter/s", "cores": 1,
                               "kind": "oracle", "variant": "O-STAGE", "cpu": _cpu_model(),
                               "host_cores": os.cpu_count(), "median_ms": med * 1e3,
                               "trials_ms": [x * 1e3 for x in secs],
                               "sample": f"{args.cpu_trials} whole O-STAGE fixpoints of {args.workload} "
                                         f"(oracle/lp_oracle.c stage_core, steady clock around the "
                                         f"fixpoint only; occurrence lists built once, untimed), "
                                         f"pinned to core {core}; {wall:.1f} s wall incl. ingest",
                               "gpu_speedup_full": med * 1e3 / ms_max}
        if "frontier" in out:
            out["cpu_baseline"]["gpu_speedup_frontier"] = med * 1e3 / out["frontier"]["ms_per_step"]
        # the oracle's plain definition (Jacobi T_P over every rule each pass) as a
        # separately labelled extra: one whole fixpoint, the same pinned core
        old_aff = os.sched_getaffinity(0)
        try:
            os.sched_setaffinity(0, {core})
            t0 = time.perf_counter()
            _, jit, _, jconv = oracle.lm_jacobi(P)
            tj = time.perf_counter() - t0
        finally:
            os.sched_setaffinity(0, old_aff)
        assert jconv and jit == iters
        out["cpu_jacobi"] = {"value": nnz * iters / tj, "unit": "nnz*iter/s", "cores": 1, "ms": tj * 1e3,
                             "kind": "oracle O-LM Jacobi (oracle/lp_oracle.c orc_lm_jacobi: every rule, every pass)",
                             "sample": f"one whole fixpoint of {args.workload}, core {core}"}
        out["model_check"] = "main-line model == oracle O-STAGE model (bit-exact), iters equal"
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
