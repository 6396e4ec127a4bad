import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank(); n = dist.get_world_size()
torch.cuda.set_device(0)
t = torch.arange(8, device="cuda", dtype=torch.bfloat16) + 10 * r
res = {}
def tryit(name, fn):
    try:
        fn(); res[name] = "ok"
    except Exception as e:
        res[name] = "ERR " + str(e)[:100]
tryit("all_gather_into_tensor", lambda: dist.all_gather_into_tensor(torch.empty(8 * n, device="cuda", dtype=torch.bfloat16), t))
tryit("all_to_all_single", lambda: dist.all_to_all_single(torch.empty_like(t), t))
tryit("reduce_scatter_tensor", lambda: dist.reduce_scatter_tensor(torch.empty(4, device="cuda"), torch.ones(4 * n, device="cuda")))
tryit("all_reduce", lambda: dist.all_reduce(torch.ones(3, device="cuda")))
tryit("async_a2a", lambda: dist.all_to_all_single(torch.empty_like(t), t, async_op=True).wait())
if r == 0:
    print(res)
dist.destroy_process_group()
