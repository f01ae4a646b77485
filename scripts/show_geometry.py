import sys
sys.path.insert(0, '.')
import bench
for w in sys.argv[1:]:
    inp = bench.build_inputs(w)
    P = inp['P']
    sim = P.Simulation(inp["grid"], inp["problem"].solver, inp["params"], inp["bspec"], limiter=inp["limiter"], initial_max_speed=inp["speed"])
    print(w, [sim.device_grid.segments(ax) for ax in range(inp['spec'].ndim)])
    sim.close()
