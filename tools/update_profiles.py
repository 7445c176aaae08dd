"""Copy a tools/gpu_refresh.sh run (gpurun_out/) into profiles/: bench line, ncu launch list +
per-kernel summary, full-capture summary of the dominant launch, and its DRAM traffic per gate.

usage: update_profiles.py ITEMS_IN_CAPTURED_LAUNCH [LABEL]"""
import csv, io, json, os, shutil, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
items = int(sys.argv[1])
label = sys.argv[2] if len(sys.argv) > 2 else "resident"
KERNEL = {"resident": "resident_tc_kernel<9,29,true,2,false>", "tiled": "level_tc_ws_kernel<9,29,true,1>"}.get(
    label, "level_tc_ws_kernel<9,29,true,2>")
RND = os.environ.get("ROUND", "r2")
FNAME = f"{RND}_ncu_full_resident" if label == "resident" else f"{RND}_ncu_full_level_tc_ws_{label}"
shutil.copy(os.path.join(G, "bench_default.json"), os.path.join(P, f"{RND}_bench_default_final.json"))
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{RND}_launches_bench_default.csv"))
rows = list(csv.reader(open(os.path.join(P, f"{RND}_launches_bench_default.csv"))))
i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[i], rows[i + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
t, c = defaultdict(float), defaultdict(int)
for r in data:
    k = r[ki].split("(")[0]
    t[k] += float(r[vi].replace(",", ""))
    c[k] += 1
tot = sum(t.values())
lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 600 python bench.py (default args)",
         "# per-kernel totals over the first 600 launches (cold-cache, serialised: shares, not absolutes)",
         "# cfg1 runs as ONE lane-resident launch per step (resident_tc_kernel); cfg4 as ONE register-file launch (regfile_tc_kernel), cfg0 as ONE warp-dataflow launch"
         " (flow_kernel), cfg2/cfg3 as ready-queue launches (level_tc_ws_kernel with the queue)",
         f"# total {tot / 1e6:.2f} ms over {len(data)} launches"]
lines += [f"{v / 1e6:10.3f} ms  {100 * v / tot:5.1f}%  n={c[k]:4d}  {k}" for k, v in sorted(t.items(), key=lambda x: -x[1])]
open(os.path.join(P, f"{RND}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
rep = os.path.join(G, "ws_full.ncu-rep")
summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True, text=True).stdout
open(os.path.join(P, f"{FNAME}.txt"), "w").write(summ)
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
hdr, unit, val = raw[0], raw[1], raw[2]


def get(name):
    j = hdr.index(name)
    return float(val[j].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit[j], 1)


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
d = {"source": f"profiles/{FNAME}.txt (ncu --set full, tools/ncu_probe.py: cfg1 netlist, "
               f"one {label} launch of {KERNEL}, {items} gate items)",
     "dram_bytes_read": rd, "dram_bytes_write": wr, "items": items, "dram_bytes_per_item": (rd + wr) / items,
     "algorithmic_bytes_per_item": 25548, "padded_ciphertext_bytes_per_item": 28224, "levels_kernel_bytes_per_item": 28107.5,
     "note": ("traffic/algorithmic = %.2f: reads %.0f B/gate, writes %.0f B/gate (%s). The level schedule "
              "moved 28,108 B/gate." % ((rd + wr) / items / 25548, rd / items, wr / items,
                                        "the pairs' inputs and outputs only: intermediates stay in shared memory"
                                        if label == "resident" else
                                        "inputs; outputs plus temporaries the L2 ring did not keep"))}
json.dump(d, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=2)
print("\n".join(lines[3:]))
print(d["note"])
