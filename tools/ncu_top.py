"""Summarise an ncu report: headline metrics + top source lines by stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "Elapsed Cycles", "Executed Ipc Active", "Issued Warp Per Scheduler", "Warp Cycles Per Issued",
        "Registers Per Thread", "DRAM Throughput", "L1/TEX Hit Rate", "Achieved Occupancy", "Issue Slots Busy",
        "Executed Instructions", "Dynamic Shared Memory Per Block")
for r in csv.reader(det.splitlines()):
    if len(r) > 4 and r[-3] in keep:
        print(f"{r[-3]:40s} {r[-1]:>16s} {r[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None; tot = 0; agg = []
for r in csv.reader(src.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            s = int(r[4]); ins = int(r[7])
        except ValueError:
            continue
        agg.append((s, ins, f, r[0], r[1].strip()[:100])); tot += s
agg.sort(reverse=True)
print("total stall samples", tot)
for s, ins, f, ln, code in agg[:n]:
    print(f"{100*s/tot:5.1f}%  inst {ins:>11}  {f}:{ln}  {code}")
