import sys, statistics
sys.path[:0] = ["."]
import torch
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import cli, _native as N
from paper_1811_01566_b200.pipeline import _to_device_obs
env = cli.preset_environment("sta-paper")
g = bm.build_graph(cli.preset_pipeline("sta-paper"))
obs = [_to_device_obs(env.next_observation()) for _ in range(3)]
torch.cuda.synchronize()
print("current raw stream", N.stream_ptr(), torch.cuda.current_stream())
for i in range(6):
    outs, t = bm.execute(g, obs[i % 3])
    print([(n, round(ms, 3)) for n, ms in t.stages], round(t.total_ms, 3))
# raw DAS time
node = g.nodes["beamform"].fn
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(); node(obs[0]); b.record(); torch.cuda.synchronize()
print("beamform op alone", a.elapsed_time(b))
