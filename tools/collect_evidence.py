#!/usr/bin/env python
"""Copy one evidence pass (tools/r02_evidence.sh output under gpurun_out/<dir>) into
profiles/ and rebuild profiles/kernel_traffic.json from the ncu raw CSVs.

usage: python tools/collect_evidence.py gpurun_out/r02c [tag]     (tag defaults to r02)
"""
import csv
import json
import os
import shutil
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
# capture name -> (kernel_traffic key, workload dims, algorithmic bytes per launch)
CAPS = {
    "c2_compose1d": ("c2:fma:k32", [1 << 26], 16 * (1 << 26)),
    "c1_compose1d": ("c1:fma:k64", [1 << 20], 16 * (1 << 20)),
    "c5_box3d": ("c5:fma:k2", [768] * 3, 16 * 768 ** 3),
    "c5f32_box3d": ("c5f32:fma:k2", [768] * 3, 8 * 768 ** 3),
    "c4_compose3d": ("c4:fma:k2", [512] * 3, 16 * 512 ** 3),
    "c3b_split2d": ("c3b:fma:k4", [16384] * 2, 16 * 16384 ** 2),
    "c3a_sep_vpass": ("c3a:fma:k32:vpass", [16384] * 2, 16 * 16384 ** 2),
    "c3a_sep_hpass": ("c3a:fma:k32:hpass", [16384] * 2, 16 * 16384 ** 2),
}


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = vals[i].replace(",", "")
        return float(v) * SCALE.get(units[i], 1.0) if v else 0.0
    return {"kernel": vals[hdr.index("Kernel Name")],
            "dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
            "lts_t_bytes": get("lts__t_bytes.sum"), "duration_us_under_ncu": get("gpu__time_duration.sum")}


def main():
    src = sys.argv[1].rstrip("/")
    tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
    prof = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    os.makedirs(os.path.join(prof, f"{tag}_ncu"), exist_ok=True)
    os.makedirs(os.path.join(prof, f"{tag}_bench_workloads"), exist_ok=True)
    shutil.copy(os.path.join(src, "bench_default.json"), os.path.join(prof, f"{tag}_bench_default.json"))
    shutil.copy(os.path.join(src, "bench_ref.json"), os.path.join(prof, f"{tag}_bench_reference_arm.json"))
    for f in sorted(os.listdir(os.path.join(src, "wl"))):
        if f.endswith(".json"):
            shutil.copy(os.path.join(src, "wl", f), os.path.join(prof, f"{tag}_bench_workloads", f))
    for name in ("launches_c5.csv", "launches_c2.csv"):
        if os.path.exists(os.path.join(src, name)):
            shutil.copy(os.path.join(src, name), os.path.join(prof, f"{tag}_{name}"))
    traffic = {"_doc": "per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each bench workload's "
                       "dominant kernel from one ncu --set full capture; key = workload:arith:k"}
    for f in sorted(os.listdir(os.path.join(src, "ncu"))):
        if f.endswith(("_summary.txt", "_stalls.txt")):
            shutil.copy(os.path.join(src, "ncu", f), os.path.join(prof, f"{tag}_ncu", f))
        if f.endswith("_raw.csv"):
            cap = f[:-len("_raw.csv")]
            if cap not in CAPS:
                continue
            key, dims, alg = CAPS[cap]
            m = raw_metrics(os.path.join(src, "ncu", f))
            m.update({"dims": dims, "traffic_bytes": m["dram_read_bytes"] + m["dram_write_bytes"],
                      "alg_bytes_per_launch": alg,
                      "source": "ncu --set full --metrics lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                f"-k regex:<kernel> -c 1 (tools/r02_evidence.sh; profiles/{tag}_ncu/{cap}_summary.txt)"})
            traffic[key] = m
    with open(os.path.join(prof, "kernel_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("collected", src, "->", prof, "; traffic keys:", [k for k in traffic if k != "_doc"])


if __name__ == "__main__":
    main()
