import sys, json, torch
sys.path.insert(0, '.')
import bench
dev = torch.device('cuda', 0)
print(json.dumps(bench.bench_configs(dev)))
print(json.dumps(bench.bench_wang(dev)))
print(json.dumps(bench.bench_configs(dev)))
