import sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_2501_03944_b200 as P
w = bench.WORKLOADS["c1"]
eng = P.Engine(bench.make_config(P, w, 1 << 40), P.SearchSpace.box(w["D"], w["lo"], w["hi"]), bench.make_objective(P, w), seed=0)
eng.initialize(); eng.enqueue(40); eng.sync()
