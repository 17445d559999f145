"""The bench job itself (BASELINE configs[1] = C2: Llama-2-7B-shaped, 32 layers,
256 ShareGPT-length requests, TD-Pipe on one stage) for an ncu DRAM-traffic
capture of its OWN kernel launches: one td_run with per-kernel timing on, then
the engine's algorithmic bytes / launches of the requested kernel class are
printed for scripts/traffic_summary.py (same launches ncu saw; the schedule is
the bench's -- C2 fits in HBM, so one prefill phase then decode; a synthetic
frozen profile replaces td_profile so that no profiling launch is captured).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:decode_attn -s SKIP -c COUNT \\
        --clock-control none --csv --log-file gpurun_out/traffic_w.csv python scripts/traffic_job.py decode_attn
    python scripts/traffic_windows.py OUT.json SKIP:gpurun_out/traffic_w.csv [...]

The per-launch algorithmic bytes (launch order) go to
gpurun_out/traffic_job_<class>_bytes.npy so that a window of ncu-captured
launches is compared with exactly the same launches.
"""
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TDPipe  # noqa: E402
from workload import SHAPES, config_workload, synthetic_profile, write_profile_csv  # noqa: E402

cls = sys.argv[1] if len(sys.argv) > 1 else "decode_attn"
wl = config_workload("C2")
csv = os.path.join(tempfile.gettempdir(), "traffic_job_profile.csv")
write_profile_csv(csv, *synthetic_profile(1024, 2048))
t = TDPipe(SHAPES["llama2_7b"], 1, device=0, profile_csv=csv)
t.submit_workload(wl)
t.td_upload()
t.td_set_timing(True)
st = t.td_run()
k = t.td_get_timing(cls)
per = t.td_get_launch_bytes(cls)
np.save(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                     f"traffic_job_{cls}_bytes.npy"), per)
t.close()
print(json.dumps({"launches": k["launches"], "algorithmic_bytes": k["bytes"], "B": "C2 job (256 requests)",
                  "mean_ctx": None, "kernel_class": cls, "generated_tokens": st["generated_tokens"],
                  "n_decode_mb": st["n_decode_mb"]}))
