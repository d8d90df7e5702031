"""Dev: per-call latency of the small configs (eager and CUDA-graph replay)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2103_10765_b200 as g
import bench
r = bench.run_small_configs(torch, g)
print(os.environ.get("GBM3D_LIB", "main"), json.dumps({k: (round(v["us_per_call"], 1), v["graph_us_per_call"] if isinstance(v["graph_us_per_call"], str) else round(v["graph_us_per_call"], 1), v["launches"]) for k, v in r.items()}))
