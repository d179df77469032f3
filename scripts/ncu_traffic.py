#!/usr/bin/env python3
"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the forward's
kernels from one `ncu --set full` capture per workload (scripts/gpu_ncu_full.sh), keyed
like bench.py's roofline breakdown -> profiles/<round>/traffic.json (read by bench.py)."""
import csv
import io
import json
import subprocess
import sys

# launch order of layer 0 in a capture of -k "gemm_|attn_tc|ln_f16|embed_f32" -c 8
LAYER_ORDER = ["embed", "ln1", "gemm_qkv", "attention", "gemm_wo", "ln2", "gemm_ffn1", "gemm_ffn2"]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k].replace(",", "")) * UNITS[units[hdr.index(k)]]
        tu = units[hdr.index("gpu__time_duration.sum")]
        t = float(d["gpu__time_duration.sum"].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(tu, 1.0)
        res.append({"kernel": d["Kernel Name"].split("(")[0], "dram_bytes": tot, "ncu_us": t})
    return res


def main(out_path, *pairs):
    table = {}
    try:  # keep the entries of workloads not re-captured this time
        with open(out_path) as f:
            table = json.load(f)
    except (OSError, ValueError):
        pass
    for spec in pairs:  # workload=layer.ncu-rep,head.ncu-rep  or  workload=small:trunk.ncu-rep,head.ncu-rep
        wl, files = spec.split("=")
        if files.startswith("small:"):  # batch-1 path: the persistent trunk kernel + the LM head
            trunk, head = files[len("small:"):].split(",")
            table[wl] = {"fwd_small": dram_bytes(trunk)[0], "gemm_head": dram_bytes(head)[0]}
            continue
        layer, head = files.split(",")
        rows = dram_bytes(layer)
        entry = {name: rows[i] for i, name in enumerate(LAYER_ORDER) if i < len(rows)}
        entry["gemm_head"] = dram_bytes(head)[0]
        if "EPI_ROWSTAT" in entry["gemm_head"]["kernel"] or "<256, 4," in entry["gemm_head"]["kernel"]:
            entry["gemm_head_nll"] = entry["gemm_head"]  # the forward+NLL step's head (bench.py key)
        table[wl] = entry
    with open(out_path, "w") as f:
        json.dump(table, f, indent=1)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:])
