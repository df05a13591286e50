"""ls_sort time per call with the launch sequence replayed from a CUDA Graph
(default) and launched directly (LS_GRAPH=0), Normal fp64 keys, same buffers
each call (the pristine input is restored by an untimed D2D copy). One JSON
line per (n, mode)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2107_03290_b200 as ls  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100000,1000000,10000000,200000000")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    s = torch.cuda.Stream()
    for n in [int(x) for x in a.sizes.split(",")]:
        src = torch.empty(n, dtype=torch.float64, device="cuda")
        datagen.Plan("normal", n, 3).device(src)
        t = torch.empty_like(src)
        ws = ls.workspace(n, ls.LS_F64)
        for mode in ("0", "1"):
            os.environ["LS_GRAPH"] = mode
            ms = []
            for r in range(a.reps + 3):
                with torch.cuda.stream(s):
                    t.copy_(src)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    ls.ls_sort(t, ws=ws, stream=s)
                    e1.record(s)
                s.synchronize()
                if r >= 3:
                    ms.append(e0.elapsed_time(e1))
            ms.sort()
            print(json.dumps({"n": n, "graph": mode == "1", "ms_median": round(ms[len(ms) // 2], 4),
                              "ms_min": round(ms[0], 4),
                              "gkeys_per_s": round(n / ms[len(ms) // 2] / 1e6, 3)}), flush=True)
        del src, t, ws
        torch.cuda.empty_cache()
    os.environ.pop("LS_GRAPH", None)


if __name__ == "__main__":
    main()
