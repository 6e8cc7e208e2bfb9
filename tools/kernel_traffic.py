"""Collect the DRAM traffic of the bench kernel leg per (dtype, shape) from ncu --set full
captures into profiles/ncu_kernel_traffic_r02.json (bench.py reads it for roofline.traffic).
python tools/kernel_traffic.py out.json rep1.ncu-rep:f64:2048x2048x2048 ..."""
import csv
import json
import subprocess
import sys

out = {}
for spec in sys.argv[2:]:
    path, dt, shape = spec.split(":")
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, data))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
              "s": 1e3, "second": 1e3}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[u["dram__bytes_write.sum"]]
    ms = float(d["gpu__time_duration.sum"].replace(",", "")) * tscale[u["gpu__time_duration.sum"]]
    out[f"{dt} {shape}"] = {"kernel": d.get("Kernel Name", "")[:120], "dram_read_bytes": rd,
                            "dram_write_bytes": wr, "traffic_bytes": rd + wr, "ncu_ms": ms,
                            "sm_ghz": float(d["sm__cycles_elapsed.avg.per_second"].replace(",", "")) *
                            {"hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1.0}[
                                u["sm__cycles_elapsed.avg.per_second"].lower()],
                            "tensor_pipe_pct": float(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]),
                            "source": path.split("/")[-1]}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
