"""Scalable generate_workload: the reference's own synth_graph(seed 7, N) for N up
to 100k; our generator (one batched K5 validation scan) vs the reference's O(N^2) scan, timed
on the host (the reference only at sizes it finishes; its time grows ~N^2)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2511_01633_b200 as glmx  # noqa: E402
from paper_2511_01633_b200.retrieve import generate_workload  # noqa: E402

for N in [int(x) for x in (sys.argv[1:] or ["2000", "5000", "20000", "100000"])]:
    rg = oracle.RefGraph(synth=(7, N))
    path = f"/tmp/wl_synth_{N}.jsonl"
    rg.save(path)
    g = glmx.PropertyGraph.load(path, device=0)
    t0 = time.perf_counter()
    got, scan_ms = generate_workload(g, 7, 1024, 0.5)
    t_ours = time.perf_counter() - t0
    row = {"nodes": N, "questions": 1024, "ours_s": t_ours, "ours_scan_ms": scan_ms}
    if N <= 5000:
        t0 = time.perf_counter()
        want = rg.generate_workload(7, 1024, 0.5)
        row["reference_s"] = time.perf_counter() - t0
        row["identical"] = got == want
    print(json.dumps(row), flush=True)
