"""Dev tool: copy the evidence tools/collect_profiles.sh left in gpurun_out/ into profiles/
(bench lines, launch lists, ncu text pages, column subsets of the raw pages) and refresh the
DRAM bytes in profiles/traffic.json from the captures."""
import csv
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
O, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

for f in ["r02_bench_default.jsonl", "r02_bench_reference.jsonl", "r02_bench_cfg1.json", "r02_bench_cfg3.json",
          "r02_bench_cfg4.json", "r02_launches_bench_cfg2.csv", "r02_launches_bench_cfg5.csv", "r02_launches_cfg2.csv",
          "r02_launches_cfg3.csv", "r02_launches_cfg5.csv", "r02_ncu_cfg2_pw16.txt", "r02_ncu_cfg3_pw16.txt",
          "r02_ncu_cfg5_wide_paired.txt"]:
    shutil.copy(os.path.join(O, f), os.path.join(P, f))
shutil.copy(os.path.join(O, "r02_ncu_cfg5_wide.txt"), os.path.join(P, "r02_ncu_cfg5_wide_final.txt"))

keep = list(csv.reader(open(os.path.join(P, "r02_ncu_cfg2_pw16_raw_subset.csv"))))[0]
traffic = json.load(open(os.path.join(P, "traffic.json")))
KEYS = {"r02_ncu_cfg2_pw16": "gemm_tc dd->dd 256x512x256 x64", "r02_ncu_cfg3_pw16": "gemm_tc dd->dd 1024x1024x1024 x16",
        "r02_ncu_cfg5_wide": "gemm_tc dd->dd 8192x8192x8192 x1", "r02_ncu_cfg5_wide_paired": "gemm_tc dd->dd 8192x16384x8192 x1"}
for src, key in KEYS.items():
    rows = list(csv.reader(open(os.path.join(O, src + "_raw.csv"))))
    h = rows[0]
    idx = [h.index(k) for k in keep if k in h]
    dst = "r02_ncu_cfg5_wide_final" if src == "r02_ncu_cfg5_wide" else src
    with open(os.path.join(P, dst + "_raw_subset.csv"), "w", newline="") as f:
        w = csv.writer(f)
        for r in rows:
            w.writerow([r[i] for i in idx])

    def val(name):
        i = h.index(name)
        return float(rows[2][i].replace(",", "")) * UNIT[rows[1][i]]
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    traffic[key].update({"dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr})
    ti = h.index("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active")
    print(f"{key}: {rows[2][h.index('gpu__time_duration.sum')]} {rows[1][h.index('gpu__time_duration.sum')]}, DRAM "
          f"{(rd + wr) / 1e9:.3f} GB ({(rd + wr) / traffic[key]['algorithmic_bytes_per_launch']:.2f}x algorithmic), tensor pipe {rows[2][ti]} %")
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
