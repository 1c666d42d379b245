"""Per-kernel share of each bench phase from an ncu launch list (the `--metrics gpu__time_duration.sum`
pass of one C3 step), written to profiles/ncu_kernel_share.json for bench.py's dominant-kernel
roofline: python tools/kernel_share.py profiles/<launches>.csv [recurrence-label]

The launch list is cold-cache and serialised, so only the SHARES are used: bench.py multiplies a
kernel's share of its phase by the phase time it measures live (CUDA events in the step's graph)."""
import collections
import csv
import json
import os
import sys

PHASE_OF = {  # kernel-name prefix -> bench phase
    "gemm_tc1s_kernel<4, EpiB1IO": "bwd_rec", "gemm_tc1s_kernel<4, EpiB2": "bwd_rec",
    "gemm_tc_kernel<64, EpiB2": "bwd_rec", "bwd_recur_kernel": "bwd_rec",
    "gemm_tc1s_kernel<4, EpiF1IO": "fwd_rec", "gemm_tc2_kernel<256, EpiF2IO": "fwd_rec", "fwd_recur_kernel": "fwd_rec",
    "gemm_tc2_kernel<512, EpiWgrad": "wgrad", "gemm_tc1s_kernel<4, EpiWgrad": "wgrad", "seg_gemm_kernel": "wgrad",
    "seg_finalize_kernel": "wgrad", "db_kernel": "wgrad",
    "gemm_tc2p_kernel<256, EpiY": "decoder",
}


def short(name):
    n = name.replace("void ", "").replace("mlstm::", "")
    n = n.split("(CUtensorMap")[0].split("(Net")[0].split("(const")[0]
    return n.replace("<__half>", "").replace(", 0>", ">").replace(", 1>", ",MN>").replace(", 2>", ",BMN>").replace(" ", "")


def main():
    src = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else "per_timestep"
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].replace("void ", "").replace("mlstm::", "")
        phase = next((ph for k, ph in PHASE_OF.items() if name.startswith(k)), None)
        if phase is None:
            continue
        a = agg[(phase, short(d["Kernel Name"]))]
        a[0] += 1
        a[1] += float(d["Metric Value"])
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_kernel_share.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    tab = {}
    for (ph, k), (n, ns) in agg.items():
        tot = sum(v[1] for (p2, _), v in agg.items() if p2 == ph)
        tab.setdefault(ph, {})[k] = {"launches": n, "share": round(ns / tot, 4), "ncu_us_per_launch": round(ns / n / 1e3, 2)}
    out["_doc"] = ("share of each bench phase's kernel time per kernel and launches per step, from the ncu launch "
                   "list named in `source` (cold-cache, serialised: used for shares only)")
    out[label] = {"source": os.path.relpath(src), "phases": tab}
    json.dump(out, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(out[label], indent=1))


if __name__ == "__main__":
    main()
