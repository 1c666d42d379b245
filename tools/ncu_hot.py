"""Top stall lines of an ncu report: python tools/ncu_hot.py rep.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
for w in ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]:
    if w in h:
        print(f"  {w} = {v[h.index(w)]} {r[1][h.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
key = "Warp Stall Sampling (All Samples)"


def _num(v):
    try:
        return float(v or 0)
    except ValueError:
        return None


data = [dict(zip(hdr, x)) for x in rows[2:] if len(x) == len(hdr)]
data = [d for d in data if key in d and _num(d[key]) is not None]
tot = sum(float(d[key] or 0) for d in data)
for d in sorted(data, key=lambda d: -float(d[key] or 0))[:n]:
    print(f"{float(d[key]) / tot * 100:5.1f}%  {d['Source'][:100]}  exec={d['Instructions Executed']}")
