"""Probe: iterations to the stagnation stop and the fast-mode trajectory per config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2605_01748_b200 as pf

for name in sys.argv[1:]:
    topo, tab, flat = bench.build_inputs(name)
    inst = pf.build_instance_flat(topo, tab, flat, device=0)
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    t = time.time()
    done = s.run(5000)
    r = s.result()
    rates, sums = s.finish()
    print(name, inst.num_pairs, "iterations", r.iterations, "alpha", r.alpha, "converged", r.converged,
          "loop_ms", round(r.loop_ms, 1), "proj_ms", round(r.projection_ms, 1), "wall", round(time.time() - t, 2),
          flush=True)
