"""Does the runtime's CUDA-graph capture survive real NCCL collectives on its streams?
One process, NCCL world of 1: the exchange runs a genuine all_gather_into_tensor (NCCL) on the
VQ side stream inside the captured graph, then replicates the payload into the other
simulated ranks' slots (loopback), for a rank of an N=4 split.  Checks graph replay == eager."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_19342_b200 import cluster, data, model, vq  # noqa: E402
from paper_2505_19342_b200.runtime import AstraRuntime  # noqa: E402


class NcclLoopback:
    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def all_gather(self, out, inp):
        n = inp.numel()
        dist.all_gather_into_tensor(out.view(-1)[:n], inp.view(-1))   # real NCCL (1 rank)
        out.view(self.world, -1)[1:].copy_(out.view(self.world, -1)[:1].expand(self.world - 1, -1))

    def broadcast(self, t, src):
        dist.broadcast(t, src=0)


os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = model.ModelConfig(layers=4, hidden=768, heads=12, vocab_or_classes=1000, max_tokens=197,
                        causal=False, codebook_size=1024, groups=1)
params = model.init_params(cfg, seed=0)
xs = data.make_classify_batch(768, 196, 16, seed=1)
rng = np.random.default_rng(0)
flat = xs.reshape(-1, 768)
for i, b in enumerate(params.blocks):
    b.codebook = vq.Codebook(layer_id=i, groups=1, centroids=[flat[rng.choice(len(flat), 1024, replace=False)]])
plan = cluster.partition_tokens(196, 4)
rt = AstraRuntime(params, plan, batch=16, precision="fast", comm=NcclLoopback(3, 4))
x_local = np.ascontiguousarray(xs)
rt.stage_input(x_local)
rt.forward()
torch.cuda.synchronize()
eager = rt.logits.clone()
rt.capture(warmup=1)
rt.run()
torch.cuda.synchronize()
graph = rt.logits.clone()
err = (graph - eager).abs().max().item()
print(f"NCCL-in-graph capture ok: replay vs eager max |diff| = {err:.3e}")
assert err == 0.0
st, sp = plan.ranges[3]
out = rt.classify_stream([torch.from_numpy(np.ascontiguousarray(x_local[:, st:sp])).pin_memory()] * 3)
print("classify_stream ok", out[0].shape)
dist.destroy_process_group()
