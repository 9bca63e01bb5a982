"""Device vs host time per PGX env call (sample / step_), C4 at 2^22 envs."""
import time, torch, json, sys
sys.path.insert(0, '.')
import paper_2506_22609_b200 as lx
env = lx.LudaxEnvironment("connect_four", auto_reset=True)
B = 1 << 22
st = env.init(seed=1, batch_size=B)
for _ in range(5):
    st = env.step_(st, env.random_actions(st))
torch.cuda.synchronize()
# device time of 50 back-to-back samples (pure: state unchanged)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dev_sample = []
for rep in range(8):
    e0.record()
    for _ in range(50):
        a = env.random_actions(st)
    e1.record(); torch.cuda.synchronize()
    dev_sample.append(round(e0.elapsed_time(e1) / 50, 4))
# host time per call
t0 = time.perf_counter()
for _ in range(50):
    a = env.random_actions(st)
host_sample = (time.perf_counter() - t0) / 50 * 1e3
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    st = env.step_(st, a)
host_step = (time.perf_counter() - t0) / 50 * 1e3
torch.cuda.synchronize()
print(json.dumps({"dev_sample_ms": dev_sample, "host_sample_ms": host_sample, "host_step_ms": host_step}))
