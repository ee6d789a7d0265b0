import sys, torch
sys.path.insert(0, '.')
import bench, paper_2602_23592_b200 as kb
cfg = bench.CONFIGS['c4']
lay, q = bench.workload(cfg, 20250807)
g = lambda: torch.cuda.mem_get_info()[0] / 1e9
print('start free', g(), 'total', torch.cuda.mem_get_info()[1] / 1e9)
ctx = kb.Context(cfg['L'], cfg['H'], cfg['d'], cfg['mlp'], cfg['V'], 20250807, kb.FAST)
print('ctx', g())
ctx.model_init()
print('weights', g())
ctx.memory_compute_layout(lay, tier=kb.TIER_HOST)
print('memory', g(), ctx.memory_stats())
ctx.trim()
print('trim', g())
