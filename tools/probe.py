import os, json, torch, subprocess
p = torch.cuda.get_device_properties(0)
d = {"name": p.name, "sms": p.multi_processor_count, "l2": getattr(p, "L2_cache_size", None),
     "mem": p.total_memory, "cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
     "cc": [p.major, p.minor]}
print(json.dumps(d))
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.limit", "--format=csv"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500])
