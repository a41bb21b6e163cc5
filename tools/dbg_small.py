import sys; sys.path.insert(0,'.')
import workloads as W
from paper_2505_14538_b200 import Context
p = W.lattice(4, h_factor=1.0)
print(p['h'][:3], p['h'].min(), p['h'].max())
try:
    c = Context(p); print("created!", c.counters())
except Exception as e: print("raised", e)
