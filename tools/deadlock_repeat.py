import sys, json, subprocess, torch
sys.path.insert(0, '.')
import bench
dev = torch.device('cuda:0')
for i in range(6):
    o = bench.bench_deadlock(dev)
    clk = subprocess.run(['nvidia-smi','--query-gpu=clocks.sm','--format=csv,noheader'],capture_output=True,text=True).stdout.strip()
    print(i, {k: round(v['us_per_shell'],2) for k,v in o.items()}, clk, flush=True)
