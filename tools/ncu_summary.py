"""Summarise an ncu report: key metrics + SASS hot regions (split at sync/tensor ops)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
hdr = det[0]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Eligible Warps Per Scheduler", "No Eligible", "L2 Hit Rate", "Compute (SM) Throughput")
for row in det[1:]:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:32s} {d['Metric Value']:>16s} {d.get('Metric Unit','')}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
if len(raw) > 2:
    rh = raw[0]
    rv = raw[2] if len(raw) > 2 else raw[1]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
        for i, h in enumerate(rh):
            if h.startswith(k):
                print(f"{h:70s} {raw[1][i]:>8s} {rv[i]}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv"))))
h = src[1]; data = src[2:]
ie = h.index("Instructions Executed"); ss = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie]) for r in data) or 1; tots = sum(int(r[ss]) for r in data) or 1
print("total warp instr", tot, "stall samples", tots)
marks = [i for i, r in enumerate(data) if any(k in r[1] for k in
         ("UTC", "STTM", "LDTM", "SYNCS", "UBLKCP", "BAR.SYNC", "SHFL"))]
b = [0] + marks + [len(data)]
for x, y in zip(b[:-1], b[1:]):
    ins = sum(int(r[ie]) for r in data[x:y]); smp = sum(int(r[ss]) for r in data[x:y])
    if ins > 0.015 * tot or smp > 0.015 * tots:
        print(f"[{x:5d},{y:5d}) instr {ins/tot*100:5.1f}%  stall-samples {smp/tots*100:5.1f}%  {data[x][1].strip()[:50]}")
