"""Summarise ncu outputs into profiles/*.md (launch list shares; full-capture key metrics)."""
import collections, csv, subprocess, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    tot, cnt = collections.Counter(), collections.Counter()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "nsecond"), 1e-3)
        name = d["Kernel Name"].split("(")[0][:80]
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"launches: {sum(cnt.values())}, total device time {T/1e3:.1f} ms (cold-cache, serialised under ncu)", "",
           "| share | total us | launches | avg us | kernel |", "|---:|---:|---:|---:|---|"]
    for n, v in tot.most_common(20):
        out.append(f"| {v/T*100:.2f}% | {v:.1f} | {cnt[n]} | {v/cnt[n]:.2f} | `{n}` |")
    mine = {n: v for n, v in tot.items() if "p3::" in n}
    out.append("")
    out.append("libp3 kernels: " + ", ".join(f"`{n}` {v/T*100:.2f}% ({cnt[n]} launches, avg {v/cnt[n]:.1f} us)" for n, v in mine.items()))
    return "\n".join(out)

def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_bytes.sum"]
    out = ["| metric | value | unit |", "|---|---:|---|"]
    for k in keys:
        if k in d:
            out.append(f"| `{k}` | {d[k]} | {u.get(k, '')} |")
    return "\n".join(out)

if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
