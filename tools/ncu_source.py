"""Per-instruction stall samples from an ncu report's source page (SASS).

    python tools/ncu_source.py prof.ncu-rep KERNEL_SUBSTRING [--top 40] [--range 0xA-0xB]
Prints the stall-reason totals for the kernel, then the instructions with the most samples
(with their dominant reasons) in address order.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, sub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name",')
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if sub not in name:
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        hdr = rows[0]
        ia, isrc, isamp, iexec = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = {hdr[i]: 0 for i in stall_cols}
        recs = []
        base = None
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            addr = int(r[ia], 16)
            base = addr if base is None else base
            s = int(r[isamp] or 0)
            reasons = {hdr[i]: int(r[i] or 0) for i in stall_cols}
            for k, v in reasons.items():
                tot[k] += v
            recs.append((addr - base, r[isrc].strip(), s, int(r[iexec] or 0), reasons))
        allsamp = sum(x[2] for x in recs)
        print(f"== {name[:100]}  samples={allsamp}")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            if v:
                print(f"   {k:24s} {v:8d} {100.0 * v / max(1, allsamp):5.1f}%")
        hot = sorted(recs, key=lambda x: -x[2])[:top]
        hot.sort()
        for off, src, s, ex, reasons in hot:
            rs = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
            print(f"  {off:#07x} {s:7d} ex={ex:10d} {src[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in rs if v))


if __name__ == "__main__":
    main()
