"""Host-pipeline chunk-count sweep: the e2e call (pinned host buffers, H2D +
merge + D2H) of one BASELINE config at the chunk counts given, one process per
count (COMERGE_HOST_CHUNKS is read once per process).

    python tools/e2e_chunks.py C4 8 16 32 64
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, ROOT)
    import torch
    import bench
    cfg = sys.argv[2]
    inp = bench.make_inputs(cfg, device=torch.device("cuda:0"))
    r = bench.e2e_measure(cfg, inp, 7, 2)
    print(f"{cfg} chunks={os.environ.get('COMERGE_HOST_CHUNKS', 'default')} "
          f"e2e {r['ms_per_step']:.2f} ms  {r['value'] / 1e9:.3f} G elem/s  calls ms "
          f"{[round(x, 2) for x in r.get('calls_ms', [])]} cpu {__import__("ctypes").CDLL(None).sched_getcpu()}", flush=True)
    sys.exit(0)

cfg = sys.argv[1]
for k in sys.argv[2:]:
    env = dict(os.environ)
    if k != "default":
        env["COMERGE_HOST_CHUNKS"] = k
    subprocess.run([sys.executable, os.path.abspath(__file__), "--one", cfg], env=env, check=False)
