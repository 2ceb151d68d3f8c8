import os, sys
sys.path.insert(0, os.getcwd())
import paper_1603_06400_b200 as P
from workloads import make_config
for ci in (1, 2):
    G = P.Geometry(make_config(ci).desc())
    print(ci, G.query("esai_breakpoints"), G.query("esai_max_window"), G.query("esai_window_permille"), G.query("esai_tile_span_permille"))
