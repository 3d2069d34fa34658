"""Warp-stall samples of one layer_kernel capture, split by kernel region.

    python tools/source_regions.py gpurun_out/X_src_sass.csv [out.json]

Input: `ncu -i X.ncu-rep --page source --csv --print-source sass` of a capture
taken with `--set full --import-source on`. The regions are found from the
SASS itself (no hard-coded addresses): the consumer record loop is the span
from the first to the last FFMA2 of the mask loop; the consumer entry wait is
the mbarrier try-wait loop right before it; everything before that belongs to
the producer and publisher warps, everything after it to the consumers'
epilogue and unit bookkeeping.
"""
import csv
import json
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    addr = [int(r[0], 16) for r in data]
    src = [r[1] for r in data]
    ffma = [i for i, s in enumerate(src) if "FFMA2" in s]
    lo, hi = ffma[0], ffma[-1]
    # the consumer's entry wait: the last try-wait before the loop
    wait = max(i for i in range(lo) if "TRYWAIT" in src[i])
    # consumer section starts a few instructions before its wait (the
    # S2UR of the shared window base the wait address is built from)
    start = max(i for i in range(wait) if "S2UR" in src[i] and "CgaCtaId" in src[i])
    regions = {
        "producer+publisher": range(0, start),
        "consumer: entry wait + unit setup": range(start, lo),
        "consumer: record loop": range(lo, hi + 1),
        "consumer: epilogue + bookkeeping": range(hi + 1, len(data)),
    }
    total = sum(int(r[ix["# Samples"]]) for r in data)
    res = {"source": path, "total_samples": total, "regions": {}}
    for name, rg in regions.items():
        smp = sum(int(data[i][ix["# Samples"]]) for i in rg)
        ins = sum(int(data[i][ix["Instructions Executed"]] or 0) for i in rg)
        ff = sum(int(data[i][ix["Instructions Executed"]] or 0) for i in rg if "FFMA2" in src[i])
        top = {s[6:]: sum(int(data[i][ix[s]]) for i in rg) for s in stalls}
        top = dict(sorted(((k, v) for k, v in top.items() if v), key=lambda kv: -kv[1])[:5])
        res["regions"][name] = {"samples": smp, "share": round(smp / total, 4),
                                "warp_instructions": ins, "ffma2": ff, "top_stalls": top}
    cons = sum(v["samples"] for k, v in res["regions"].items() if k.startswith("consumer"))
    for k, v in res["regions"].items():
        if k.startswith("consumer"):
            v["share_of_consumer_time"] = round(v["samples"] / cons, 4)
    text = json.dumps(res, indent=1)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
