"""Per-kernel timeline of one C3 train step from the in-kernel %globaltimer trace."""
import os, sys, collections
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_1808_01371_b200 as M
from synth import bytestream
h, e, B, T = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 64, 256, 256)))
cfg = M.mlstm_default_config(hidden=h, embed=e, batch=B, seq_len=T)
m = M.MLSTM(cfg)
by = torch.from_numpy(bytestream.window(np.arange(B), 0, T)).cuda()
m.train_step(by); m.train_step(by)
M.mlstm_trace_enable(1 << 20)
m.train_step(by)
rec = M.mlstm_trace_read(1 << 20).astype(np.int64)
M.mlstm_trace_enable(0)
names = {1: "F1", 2: "F2", 3: "B1", 4: "B2", 5: "dec", 6: "dHdec", 7: "tab", 8: "wgrad", 9: "partial"}
t0 = rec[:, 2].min()
# group CTAs into launches: consecutive records of the same tag whose start times overlap
rec = rec[np.argsort(rec[:, 2])]
launches = []
for r in rec:
    if launches and launches[-1]["tag"] == r[0] and r[2] <= launches[-1]["end"] + 500:
        L = launches[-1]
    else:
        L = {"tag": r[0], "rows": [], "end": 0}
        launches.append(L)
    L["rows"].append(r)
    L["end"] = max(L["end"], r[7])
stats = collections.defaultdict(list)
prev_end = None
for L in launches:
    R = np.array(L["rows"])
    st, en = R[:, 2].min(), R[:, 7].max()
    d = lambda a, b: np.mean(np.where((R[:, a] > 0) & (R[:, b] > 0), R[:, b] - R[:, a], np.nan))
    stats[L["tag"]].append([en - st, d(2, 3), d(3, 4), d(4, 5), d(5, 6) if (R[:, 6] > 0).any() else np.nan,
                            d(6, 7) if (R[:, 6] > 0).any() else d(5, 7), (st - prev_end) if prev_end else np.nan,
                            len(R)])
    prev_end = en
R6 = rec[(rec[:, 8] > 0)]
if len(R6):
    for tag in sorted(set(R6[:, 0].tolist())):
        X = R6[R6[:, 0] == tag]
        print(f"  {names.get(tag, tag)} split-K epilogue: reduce {np.mean(X[:, 8] - X[:, 6]) / 1e3:.2f} us, "
              f"tile {np.mean(np.where(X[:, 10] > 0, X[:, 10] - X[:, 9], 0)) / 1e3:.2f} us, "
              f"after {np.mean(X[:, 7] - np.maximum(X[:, 8], X[:, 10])) / 1e3:.2f} us")
print("tag      n   span_us  start->tma  tma->data  data->acc  acc->reduced  ->end  gap_before  ctas")
for tag, v in sorted(stats.items()):
    a = np.nanmean(np.array(v, dtype=float), axis=0) / 1e3
    print(f"{names.get(tag, tag):8s} {len(v):4d} {a[0]:8.2f} {a[1]:10.2f} {a[2]:10.2f} {a[3]:10.2f} {a[4]:12.2f} "
          f"{a[5]:7.2f} {a[6]:10.2f} {a[7]*1e3:6.0f}")
print("\nper-launch (wgrad / dec / dHdec / tab):")
for L in launches:
    if L["tag"] in (5, 6, 7, 8):
        R = np.array(L["rows"])
        print(f"  {names.get(L['tag'])}: span {(R[:, 7].max() - R[:, 2].min()) / 1e3:9.1f} us, ctas {len(R)}, "
              f"mean cta {(R[:, 7] - R[:, 2]).mean() / 1e3:8.1f} us")
