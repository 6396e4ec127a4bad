"""Multi-process DAP end-to-end check with the real CUDA kernels.

    torchrun --nproc-per-node N scripts/dap_check.py      (EVO_DIST_BACKEND=gloo|nccl)

Every rank runs DapStack fwd+bwd (2 blocks, tiny config) on its shards; rank 0
compares the gathered outputs, input gradients and the all-reduced parameter
gradients with the single-device EvoformerStack, and the forward ledger with
predict_block_ledger.  With gloo, all ranks may share one GPU."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2203_00854_b200.config import EvoConfig, synthetic_inputs
from paper_2203_00854_b200.dap import CommLedger, DapComm, DapStack, predict_block_ledger
from paper_2203_00854_b200.evoformer import EvoformerStack

backend = os.environ.get("EVO_DIST_BACKEND", "gloo")
dist.init_process_group(backend)
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
cfg = EvoConfig(16, 32, 64, 32, 2, 1, 16)
m64, z64 = synthetic_inputs(cfg, 5)
rng = np.random.default_rng(6)
gm64, gz64 = rng.normal(size=m64.shape), rng.normal(size=z64.shape)
led = CommLedger(world, 2)
comm = DapComm(ledger=led)
st = DapStack(cfg, 2, seed=5, comm=comm)
m, z = st.shard_inputs(m64, z64, "cuda")
gm, gz = st.shard_inputs(gm64, gz64, "cuda")
st.zero_grad()
mo, zo, saved = st.forward(m, z)
fwd_ledger = led.summary()
comm.ledger = None
dm, dz = st.backward(saved, gm, gz)
loss = (mo.float() * gm.float()).sum() + (zo.float() * gz.float()).sum()
dist.all_reduce(loss)
full = [comm.all_gather(t).flatten(0, 1) for t in (mo, zo, dm, dz)]
torch.cuda.synchronize()
ok = True
if rank == 0:
    ref = EvoformerStack(cfg, 2, seed=5)
    ref.zero_grad()
    dev = lambda a: torch.tensor(a, device="cuda").bfloat16()
    mo1, zo1, sv1 = ref.forward(dev(m64), dev(z64))
    loss1 = (mo1.float() * dev(gm64).float()).sum() + (zo1.float() * dev(gz64).float()).sum()
    dm1, dz1 = ref.backward(sv1, dev(gm64), dev(gz64))
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm())
    errs = {"m": rel(full[0], mo1), "z": rel(full[1], zo1), "dm": rel(full[2], dm1), "dz": rel(full[3], dz1),
            "loss": abs(float(loss) - float(loss1)) / abs(float(loss1)),
            "grad": max(rel(a.grad, b.grad) for a, b in zip(st.blocks, ref.blocks))}
    want = {k: {"count": 2 * v["count"], "bytes": 2 * v["bytes"]} for k, v in predict_block_ledger(cfg, world, 2).items()}
    ok = max(errs.values()) <= 2e-2 and fwd_ledger == want
    print("DAP_CHECK", "OK" if ok else "FAIL", backend, world, errs, fwd_ledger == want, flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
