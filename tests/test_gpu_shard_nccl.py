"""The head-range-sharded least model through its public API (shard.ShardedLeastModel)
on the GPU with NCCL, one rank (the only GPU this run has): the product's per-pass loop --
one θ-pass, the NCCL all-gather of owned words + status word, the device combine, the
lag-1 flag read from mapped host memory -- against the oracle (model, pass count,
popcount trace), with start sets given as a mask and as packed words.  Runs in a
subprocess so its process group does not outlive the test."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, ROOT)
import lpgen, oracle
from paper_2009_10247_b200 import lp
from paper_2009_10247_b200.shard import ShardedLeastModel
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
for name in ("C1", "C2", "rand"):
    if name == "rand":
        P = lpgen.random_program(np.random.default_rng(3), 20000, 80000, max_len=5, n_facts=150)
    else:
        P = lpgen.config(name)
    sh = ShardedLeastModel(P)
    rng = np.random.default_rng(7)
    for start in (None, "mask", "words"):
        v0 = None if start is None else rng.choice(P.n_atoms, size=P.n_atoms // 50, replace=False)
        om, stage, oit = oracle.lm_stage(P, v0=None if v0 is None else v0.tolist())
        if start == "words":
            mask = np.zeros(P.n_atoms, dtype=bool); mask[v0] = True
            m, it, pops = sh.run(v0_words=lp.pack_mask(mask))
        elif start == "mask":
            mask = np.zeros(P.n_atoms, dtype=bool); mask[v0] = True
            m, it, pops = sh.run(v0=mask)
        else:
            m, it, pops = sh.run()
        assert it == oit, (name, start, it, oit)
        assert (m == oracle.pack_bits(om)).all(), (name, start)
        assert pops == oracle.popcounts_from_stage(stage, oit), (name, start)
        m2, it2, _ = sh.run(popcounts=False)        # (a second call on the same buffers)
    print("ok", name, oit)
dist.destroy_process_group()
'''


def test_sharded_least_model_nccl_one_rank():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device (these tests run on the B200 box)")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29593")
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count("ok ") == 3
