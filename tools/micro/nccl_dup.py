import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def run(r):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=r, world_size=2, device_id=torch.device("cuda:0"))
    t = torch.ones(4, device="cuda:0") * (r + 1)
    try:
        dist.all_reduce(t); torch.cuda.synchronize(); print("rank", r, "ok", t.tolist(), flush=True)
    except Exception as e:
        print("rank", r, "fail", repr(e)[:300], flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(run, nprocs=2)
