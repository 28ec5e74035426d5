"""Write the round's profile summaries under profiles/ from gpurun_out/
artifacts: ncu --set full reports (kernel tables + source hotspots), the
launch list of the bench command (ncu gpu__time_duration per launch) and
the bench JSON line.

usage: python tools/make_profiles.py ROUND name=REPORT.ncu-rep ... \
           [launches=LAUNCHES.csv] [bench=BENCH.json]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402


def lines(rep, top=25):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, str(top)],
                         capture_output=True, text=True).stdout
    return out


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = {}
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        if name not in per:
            order.append(name)
        per.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in per.values()) or 1
    out = ["| kernel | launches | mean ns | share of listed time |", "|---|---|---|---|"]
    for n in order:
        v = per[n]
        out.append(f"| `{n}` | {len(v)} | {sum(v)/len(v):.0f} | {100*sum(v)/tot:.1f}% |")
    return "\n".join(out)


def traffic(rep):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) per captured kernel."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(out.splitlines()))
    head, units = r[0], r[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for row in r[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        name = d["Kernel Name"].replace("void ", "").split("(")[0].replace(" ", "")
        tot = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res[name] = tot
    return res


def main():
    rnd = sys.argv[1]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    for arg in sys.argv[2:]:
        key, path = arg.split("=", 1)
        if key == "launches":
            dst = os.path.join(ROOT, "profiles", f"{rnd}_launches.csv")
            with open(path) as f, open(dst, "w") as g:
                g.write(f.read())
            with open(os.path.join(ROOT, "profiles", f"{rnd}_launches.md"), "w") as g:
                g.write(f"# {rnd}: launch list of `python bench.py --steps 3 --warmup 3 --no-cpu-baseline` under "
                        "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400`\n\n")
                g.write("Cold-cache, serialised per-launch times (ncu replay); only the kernels' "
                        "relative share is meaningful, not the absolute step time.\n\n")
                g.write(launch_table(path) + "\n")
        elif key == "bench":
            d = json.load(open(path))
            with open(os.path.join(ROOT, "profiles", f"{rnd}_bench.json"), "w") as g:
                json.dump(d, g, indent=1)
        else:
            tp = os.path.join(ROOT, "profiles", f"{rnd}_traffic.json")
            tr = json.load(open(tp)) if os.path.exists(tp) else {}
            tr.update(traffic(path))
            with open(tp, "w") as g:
                json.dump(tr, g, indent=1)
            with open(os.path.join(ROOT, "profiles", f"{rnd}_{key}.md"), "w") as g:
                g.write(f"# {rnd}: `{key}` — ncu --set full --import-source on (one launch)\n\n")
                g.write(summarise(path) + "\n")
                g.write("## Source hotspots (warp-stall samples / executed instructions)\n\n```\n")
                g.write(lines(path) + "```\n")


if __name__ == "__main__":
    main()
