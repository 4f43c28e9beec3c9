import sys, numpy as np
sys.path.insert(0, '.')
import paper_2411_11244_b200 as md
a, b = md.gen_scene("interlocked-rings", {"nu": 8, "nv": 4})
t = md.build_f12(a)
box = t._box.cpu().numpy().reshape(-1, 6)[1:]
L = t.leaf_count
def leafunion(node, lvl):
    k = t.depth - lvl
    first = ((node + 1) << k) - 1
    ls = box[first:first + (1 << k)]
    return np.concatenate([ls[:, :3].min(0), ls[:, 3:].max(0)])
for node in [11, 12, 3, 4, 23, 24, 25, 26]:
    lvl = int(np.floor(np.log2(node + 1)))
    print(node, lvl, box[node].round(4), leafunion(node, lvl).round(4))
