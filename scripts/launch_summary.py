"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) into a markdown table: per kernel, launches, share of summed
device time, mean time and mean DRAM bytes. Cold-cache, serialised: shares, not absolutes."""
import csv, collections, sys

def main(src, dst, title):
    rows = [r for r in csv.DictReader(l for l in open(src) if not l.startswith("=="))]
    per = collections.defaultdict(lambda: {"n": set(), "t": 0.0, "rd": 0.0, "wr": 0.0})
    for r in rows:
        k = r["Kernel Name"][:90] + (" grid " + r["Grid Size"] if r.get("Grid Size") else "")
        d = per[k]
        d["n"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] else 0.0
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["t"] += v * scale
        elif r["Metric Name"] == "dram__bytes_read.sum":
            d["rd"] += v * scale
        elif r["Metric Name"] == "dram__bytes_write.sum":
            d["wr"] += v * scale
    tot = sum(d["t"] for d in per.values())
    out = [f"# {title}", "", f"launches: {sum(len(d['n']) for d in per.values())}; summed device time "
           f"{tot / 1e3:.1f} us (ncu --clock-control none, cold-cache, serialised: use the shares)", "",
           "| kernel | launches | share of time | mean time (us) | mean DRAM read+write (MB) |", "|---|---|---|---|---|"]
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["t"]):
        n = len(d["n"])
        out.append(f"| `{k}` | {n} | {100 * d['t'] / tot:.1f}% | {d['t'] / n / 1e3:.2f} | {(d['rd'] + d['wr']) / n / 1e6:.2f} |")
    open(dst, "w").write("\n".join(out) + "\n")

if __name__ == "__main__":
    main(*sys.argv[1:4])
