"""Time mg_agglomerate_seeds (CUDA events on the calling stream) on holed quad
meshes (workloads/unstructured.py) of growing size; the oracle's time beside it
for the sizes it finishes quickly.  One JSON line per size."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1811_09909_b200 import agglomerate_seeds  # noqa: E402
from workloads.unstructured import holed_quad_mesh  # noqa: E402


def main():
    d = torch.device("cuda:0")
    for n, nlev in ((96, 7), (512, 7), (2048, 8)):
        m = holed_quad_mesh(n, holes=12, sx=4, sy=2, seed=9)
        ee = torch.from_numpy(m.edge_elem).to(d).contiguous()
        cx, cy = torch.from_numpy(m.cx).to(d), torch.from_numpy(m.cy).to(d)
        sd = torch.from_numpy(m.seeds).to(d)
        agglomerate_seeds(ee, cx, cy, sd, nlev)   # warm-up
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0.record()
            _, _, _, nme = agglomerate_seeds(ee, cx, cy, sd, nlev)
            t1.record()
            torch.cuda.synchronize()
            ms.append(t0.elapsed_time(t1))
        rec = {"n": n, "ne": m.ne, "nedge": m.nedge, "nseed": len(m.seeds), "nlev": nlev,
               "gpu_ms": min(ms), "macro_edges": nme}
        if n <= 512:
            from oracle import agglomerate as A
            t = time.time()
            lab, _ = A.agglomerate_levels(m.ne, m.edge_elem, m.cx, m.cy, m.seeds, nlev)
            for k in range(nlev - 1):
                A.macro_edges(lab[k], m.edge_elem)
            rec["oracle_s"] = time.time() - t
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
