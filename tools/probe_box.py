"""Step-0 box probe: device properties, VMM granularity and
latency, pinned host-link bandwidth, read-only HBM bandwidth, host RAM / cores.
Writes gpurun_out/probe.json. Not part of the product path."""
import json, os, time, subprocess
import torch

out = {}
p = torch.cuda.get_device_properties(0)
out["name"] = p.name
out["sms"] = p.multi_processor_count
out["total_mem"] = p.total_memory
out["l2"] = getattr(p, "L2_cache_size", None)
out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
try:
    out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
except Exception as e:
    out["meminfo"] = str(e)
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
except Exception as e:
    out["lscpu"] = str(e)
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:
    out["topo"] = str(e)

# VMM granularity + map latency via cuda-python
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    e, gmin = cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)
    e, grec = cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)
    out["gran_min"] = int(gmin); out["gran_rec"] = int(grec)
except Exception as ex:
    out["vmm_err"] = repr(ex)

def bw(fn, nbytes, iters=10):
    best = 1e9
    s = torch.cuda.Event(enable_timing=True); t = torch.cuda.Event(enable_timing=True)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    for _ in range(iters):
        s.record(); fn(); t.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(t) / 1e3)
    return nbytes / best / 1e9

N = 1 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
out["h2d_gbs"] = bw(lambda: d.copy_(h, non_blocking=True), N)
out["d2h_gbs"] = bw(lambda: h.copy_(d, non_blocking=True), N)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
out["bidir_gbs"] = bw(both, 2 * N)
# read-only HBM: sum over 4 GiB bf16
x = torch.empty(2 << 30, dtype=torch.bfloat16, device="cuda")
x.fill_(1.0)
out["read_sum_gbs"] = bw(lambda: x.sum(dtype=torch.float32), x.numel() * 2)
y = torch.empty_like(x)
out["copy_gbs"] = bw(lambda: y.copy_(x), x.numel() * 4)
out["free_mem"] = torch.cuda.mem_get_info()
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1, default=str)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "topo")}, default=str))
