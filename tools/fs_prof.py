import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2305_15661_b200 import fullspace
case, U, x, mu = bench._fullspace_case(25, 80)
geom = case.geom
fullspace.assemble_enriched(case.law, case.mesh, case.maps, U, x, mu, geom=geom)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
fullspace.assemble_enriched(case.law, case.mesh, case.maps, U, x, mu, geom=geom)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
