import sys, os
sys.path.insert(0, ".")
import synthdata
from paper_2312_06126_b200 import spz
h = int(sys.argv[1]); algo = sys.argv[2]
o, m = (22, 6) if algo == "sac" else (44, 17)
g = spz.Replay(o, m, 3000)
g.push(**synthdata.transitions("locomotion", o, m, 3000))
lrn = spz.Learner(g, algo=algo, precision="bf16", hidden=h, n_hidden=2, max_batch=1024, use_graph=False)
try:
    print(h, algo, lrn.update(1024, 2))
except Exception as e:
    print(h, algo, "ERR", e)
