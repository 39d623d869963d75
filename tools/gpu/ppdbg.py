import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tests"))
import numpy as np, torch
from dataclasses import replace
import paper_2603_28160_b200 as ms
from paper_2603_28160_b200 import configs, engine, planner, _native
from paper_2603_28160_b200.engine import SweepBatch
cfg, ext, _ = configs.config5()
cfg = replace(cfg, grid=ms.GridSpec.from_nodes(0.001, -0.2555, 0.0, 512, 512), edge_point_count=600)
cfg = replace(cfg, process=replace(cfg.process, initial_position_mm=(-0.2, None, 0.0)))
ext = replace(ext, passes=3, stepover_mm=0.2)
p = planner.plan(cfg, ext)
quarter = (p.grid.m + 1) * (p.grid.n + 1) * 8 // 4 + 8
engine.L2_TILE_BYTES = quarter; engine.ZCAP_L2_TILE_BYTES = quarter
def run(cuts, split=True, rejoin=False):
    b = SweepBatch([(p, 0, p.grid.n)])
    sp = _native.stream_ptr()
    b.launch_fill(sp)
    mode, jidx, _, _, _, max_pts = b.group_meta[0]
    capped = [k for k, t in enumerate(b.group_tiles[0]) if t and b.zc_seq[0][k] is not None]
    anchors = None
    for c in range(len(cuts) - 1):
        if split:
            anchors = b._launch_capped(0, capped, mode, 0, max_pts, sp, split=True, passes=(cuts[c], cuts[c+1]), anchors=None if rejoin else anchors)
            if rejoin:
                for a in anchors: _native.check(b.lib.msurf_stream_wait(sp, a))
        else:
            raise SystemExit
    for a in anchors: _native.check(b.lib.msurf_stream_wait(sp, a))
    b.launch_decode(sp)
    torch.cuda.synchronize()
    return b.heights()[0].cpu().numpy().copy()
ref = run([0, 3])
for cuts in ([0, 1, 3], [0, 2, 3], [0, 1, 2, 3], [0, 3], [0, 1, 2]):
    h = run(cuts)
    print(cuts, int(np.count_nonzero(h != ref)))
print("rejoin [0,1,2,3]", int(np.count_nonzero(run([0, 1, 2, 3], rejoin=True) != ref)))
engine.ZCAP_STAGED = False
b0 = run([0, 3])
print("unstaged [0,1,2,3] vs unstaged whole", int(np.count_nonzero(run([0, 1, 2, 3]) != b0)), "unstaged whole vs ref", int(np.count_nonzero(b0 != ref)))
print("tooth box", p.tooth_box[0], "x0", p.pass_x0)
