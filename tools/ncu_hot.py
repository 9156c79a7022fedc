"""Summarise an ncu report: SOL metrics, warp-stall hot spots with the mbarrier they wait on."""
import csv, subprocess, sys, io
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in csv.reader(io.StringIO(det)):
    if len(row) > 14 and row[-3] in ("Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
                                     "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
                                     "Achieved Occupancy"):
        print(f"{row[-3]:28s} {row[-1]:>10s} {row[-2]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
def n(x):
    try: return int(x)
    except: return 0
addr = [int(r[0], 16) for r in data]; base = addr[0]
tot = sum(n(r[iS]) for r in data)
print("samples", tot, "warp-instr", sum(n(r[iE]) for r in data))
top = sorted(range(len(data)), key=lambda i: -n(data[i][iS]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 18]
for i in top:
    j = i
    while j > 0 and 'SYNCS' not in data[j][1] and 'NANOSLEEP' not in data[j][1] and i - j < 5: j -= 1
    ctx = data[j][1].strip()[:70] if j != i else ''
    print(f"{addr[i]-base:#7x} {n(data[i][iS]):6d} {100*n(data[i][iS])/tot:5.1f}% {n(data[i][iE]):10d}  {data[i][1].strip()[:48]:48s} | {ctx}")
