"""Per-timestep timeline of the persistent dataflow recurrence (recur.cuh) from its %globaltimer trace.

usage: python tools/trace_recur.py [h B T]      (defaults: C3 = 4096 256 256)

Each CTA writes one record per timestep: tag 1000+t (forward) / 2000+u (BPTT, u = T-1-t), then
event times (ns).  Forward slots: 2 MMA F1 start, 3 first F1 block in smem, 4 F1 committed,
5 first M block in smem (F2), 6 F2 committed (MMA thread, leader CTAs); 7 F1 acc ready,
8 split-K reduced, 9 M published, 10 F2 acc ready, 11 H published (epilogue).  Backward: the same
with B1 / dA / B2 / dZ.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_01371_b200 as M  # noqa: E402
from synth import bytestream  # noqa: E402

h, B, T = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 256, 256)))
cfg = M.mlstm_default_config(hidden=h, embed=64, batch=B, seq_len=T, recurrence=1)
m = M.MLSTM(cfg)
assert m.uses_recur(), "persistent recurrence is off for this shape"
by = torch.from_numpy(bytestream.window(np.arange(B), 0, T)).cuda()
m.train_step(by)
m.train_step(by)
M.mlstm_trace_enable(1 << 20)
m.train_step(by)
rec = M.mlstm_trace_read(1 << 20).astype(np.int64)
M.mlstm_trace_enable(0)

NAMES = {
    "fwd": ["", "", "F1 start", "F1 blk0", "F1 commit", "F2 Mblk0", "F2 commit", "F1 acc", "F1 reduced",
            "M pub", "F2 acc", "H pub"],
    "bwd": ["", "", "B1 start", "B1 blk0", "B1 commit", "B2 dAblk0", "B2 commit", "B1 acc", "B1 reduced",
            "dA pub", "B2 acc", "dZ pub"],
}
for kind, base in (("fwd", 1000), ("bwd", 2000)):
    R = rec[(rec[:, 0] >= base) & (rec[:, 0] < base + T)]
    if not len(R):
        continue
    t = R[:, 0] - base
    # per timestep reference: the earliest F1/B1-accumulator-ready time over CTAs
    ref = np.array([R[t == k, 7].min() for k in range(T)])
    span = (R[:, 11].max() - R[R[:, 7] > 0, 7].min()) / 1e3
    print(f"{kind}: {len(R)} records, {R[:, 1].max() + 1} CTAs, span {span:.1f} us, "
          f"{span / T:.2f} us per timestep")
    per = np.diff(ref)
    print(f"  timestep period (median over t of consecutive F1-acc minima): {np.median(per) / 1e3:.2f} us")
    print("  event (median over CTAs and t>=2 of time relative to that timestep's first acc-ready):")
    sel = t >= 2
    for slot in range(2, 12):
        v = R[sel, slot]
        ok = v > 0
        rel = (v[ok] - ref[t[sel][ok]]) / 1e3
        if len(rel):
            print(f"    {NAMES[kind][slot]:12s} median {np.median(rel):8.2f}  p10 {np.percentile(rel, 10):8.2f}"
                  f"  p90 {np.percentile(rel, 90):8.2f} us")
    # detail records (tag base + 4000 + t): epilogue sub-phases
    dbase = base + 4000
    D = rec[(rec[:, 0] >= dbase) & (rec[:, 0] < dbase + T)]
    DN = {"fwd": {2: "F1 red: slices stored", 3: "F1 red: own+release", 4: "F1 red: peers seen", 5: "F1 red: summed",
                  6: "F2 epi: gates done", 7: "F2 epi: H stored", 8: "F2 epi: stash done"},
          "bwd": {2: "B1 red: slices stored", 3: "B1 red: own+release", 4: "B1 red: peers seen", 5: "B1 red: summed",
                  6: "B2 red: slices stored", 7: "B2 red: own+release", 8: "B2 red: peers seen", 9: "B2 red: summed",
                  10: "B2 epi: dZ stored", 11: "B2 epi: g0 loaded+math"}}[kind]
    if len(D):
        td = D[:, 0] - dbase
        sel = td >= 2
        print("  epilogue detail (same reference):")
        for slot, nm in DN.items():
            v = D[sel, slot]
            ok = v > 0
            rel = (v[ok] - ref[td[sel][ok]]) / 1e3
            if len(rel):
                print(f"    {nm:24s} median {np.median(rel):8.2f}  p10 {np.percentile(rel, 10):8.2f}"
                      f"  p90 {np.percentile(rel, 90):8.2f} us")
    # k-blocks of the sampled timestep (kRcTraceStep = 8): when each was issued / landed
    bt = base + 2000
    Bk = rec[(rec[:, 0] >= bt) & (rec[:, 0] < bt + 500)]
    if len(Bk):
        ks = 8 if kind == "fwd" else 8
        r0 = ref[ks]
        i = Bk[:, 0] - bt
        print(f"  k-blocks of timestep {ks} (times rel. to its first acc-ready; latency = full - max(w, a) issue):")
        print("    blk   w_issue   a_issue      full   latency  a_iss_cyc a_wait_cyc w_iss_cyc w_wait_cyc"
              "  (medians over CTAs; full: leader CTAs)")
        for k in sorted(set(i.tolist())):
            X = Bk[i == k]
            w, a_, f = X[:, 2], X[:, 3], X[:, 4]
            fo = f > 0
            lat = np.median((f[fo] - np.maximum(w[fo], a_[fo])) / 1e3) if fo.any() else np.nan
            print(f"    {k:3d} {np.median((w - r0) / 1e3):9.2f} {np.median((a_ - r0) / 1e3):9.2f} "
                  f"{np.median((f[fo] - r0) / 1e3) if fo.any() else np.nan:9.2f} {lat:9.2f} "
                  f"{np.median(X[:, 5]):10.0f} {np.median(X[:, 6]):9.0f} {np.median(X[:, 7]):10.0f} "
                  f"{np.median(X[:, 8]):9.0f}")
m.close()
