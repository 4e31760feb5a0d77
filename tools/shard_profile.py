"""Host / device time per pass of the head-range-sharded least model on ONE rank
(profiling aid; NCCL with world size 1).

usage: python tools/shard_profile.py [C4]
Prints, per pass, the host time of each step (the pass launch, the all-gather, the combine,
the wait for the previous pass's flag) and the device time between events around them."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
from paper_2009_10247_b200.shard import ShardedLeastModel  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29577")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
P = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
sh = ShardedLeastModel(P)
for _ in range(3):
    sh.run(popcounts=False)
torch.cuda.synchronize()
b = sh.backend
st = torch.cuda.current_stream()
rows = []
sh.v[0].copy_(sh.facts_words)
b.reset()
torch.cuda.synchronize()
T0 = time.perf_counter()
k = 0
evs = []
while True:
    v, v_next = sh.v[k & 1], sh.v[(k + 1) & 1]
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = [time.perf_counter()]
    e[0].record(st)
    b.one_pass(0, v, sh.payload)
    e[1].record(st)
    t.append(time.perf_counter())
    dist.all_gather_into_tensor(sh.gathered, sh.payload)
    e[2].record(st)
    t.append(time.perf_counter())
    b.combine(k, sh.gathered, v, v_next)
    e[3].record(st)
    t.append(time.perf_counter())
    done = k >= 1 and not b.changed(k - 1)
    t.append(time.perf_counter())
    rows.append(t)
    evs.append(e)
    if done:
        break
    k += 1
torch.cuda.synchronize()
T1 = time.perf_counter()
print(f"passes {k + 1} (iters {k}), wall {1e3 * (T1 - T0):.3f} ms")
for i, (t, e) in enumerate(zip(rows, evs)):
    print(f"pass {i:2d}: host launch {1e6 * (t[1] - t[0]):6.1f}  allgather {1e6 * (t[2] - t[1]):6.1f}  "
          f"combine {1e6 * (t[3] - t[2]):6.1f}  wait {1e6 * (t[4] - t[3]):7.1f} us | device pass "
          f"{1e3 * e[0].elapsed_time(e[1]):7.1f}  gather {1e3 * e[1].elapsed_time(e[2]):6.1f}  "
          f"combine {1e3 * e[2].elapsed_time(e[3]):6.1f} us")

# the bench's step shape: L2 flush on a side stream, barrier, events around run()
side = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for label, do_flush, do_barrier in (("plain", False, False), ("flush", True, False), ("barrier", False, True),
                                    ("flush+barrier", True, True)):
    ts = []
    for i in range(6):
        if do_flush:
            with torch.cuda.stream(side):
                flush.fill_(i)
            side.synchronize()
        if do_barrier:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sh.run(popcounts=False)
        e1.record()
        torch.cuda.synchronize()
        if i >= 1:
            ts.append(e0.elapsed_time(e1))
    print(f"run() {label:14s}: {np.mean(ts):.3f} ms (min {np.min(ts):.3f})")
dist.destroy_process_group()
