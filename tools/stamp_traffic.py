"""Write profiles/sweep_traffic.json from an `ncu --set full` capture of the
main sweep launch, stamped with the SHA-256 of the main sweep kernel's SASS in
the built library, so bench.py reports it only while that machine code is
unchanged.

    python tools/stamp_traffic.py gpurun_out/r2_sweep.ncu-rep 4 1 "<how it was captured>"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, config, ngpu, how = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                      "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
units, data = rows[0], rows[1:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
main = max(data, key=lambda r: float(r["gpu__time_duration.sum"]))
rd = float(main["dram__bytes_read.sum"]) * scale[units["dram__bytes_read.sum"]]
wr = float(main["dram__bytes_write.sum"]) * scale[units["dram__bytes_write.sum"]]
doc = {
    "config": config, "n_gpus": ngpu,
    "kernel": main["Kernel Name"].split("(")[0],
    "sweep_sass_sha256": bench._sweep_source_hash(),
    "bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
    "duration_ms": float(main["gpu__time_duration.sum"]),
    "fp64_pipe_active_pct": float(main["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
    "note": "writes are the per-source-group partial sums (2 doubles per row per group) that make row "
            "sums independent of the row split; reads are the 80-byte source records and the targets",
    "source": how,
}
json.dump(doc, open(os.path.join(ROOT, "profiles", "sweep_traffic.json"), "w"), indent=1)
print(json.dumps(doc, indent=1))
