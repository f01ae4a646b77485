import sys, torch, time
sys.path.insert(0,'.')
import bench
inp = bench.build_inputs('sw8192')
P = inp['P']
sim = P.Simulation(inp["grid"], inp["problem"].solver, inp["params"], inp["bspec"], limiter=inp["limiter"], initial_max_speed=inp["speed"], device=0)
dev = sim.device_grid
stream = torch.cuda.current_stream()
dev.set_stream(stream.cuda_stream)
for _ in range(3): sim.attempt_step()
torch.cuda.synchronize()
dt = sim.estimate_dt()[0]
print('dt', dt, 'cur', sim._cur, sim._scratch)
for ax in range(2):
    r0 = torch.cuda.Event(enable_timing=True); r1 = torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter()
    r0.record(stream)
    for _ in range(4): dev.sweep_async(ax, dt, sim._cur, sim._scratch[0], 0)
    r1.record(stream); r1.synchronize()
    print('axis', ax, 'events ms', r0.elapsed_time(r1)/4, 'wall', (time.perf_counter()-t0)/4*1e3, dev.fetch(1))
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(4): dev.sweep_async(ax, dt, sim._cur, sim._scratch[0], 0)
    torch.cuda.synchronize()
    print('  wall synced', (time.perf_counter()-t0)/4*1e3)
