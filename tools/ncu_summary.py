"""Summaries of ncu output for profiles/: (1) launch list (gpu__time_duration.sum CSV log) -> per-kernel
totals and shares; (2) `--set full` report (raw CSV from `ncu -i X --page raw --csv`) -> one line per
launch with duration, SM clock, tensor-pipe activity, DRAM bytes, L2 hit rate, registers, grid.
usage: python tools/ncu_summary.py launches <launches.csv> <title>
       python tools/ncu_summary.py full <raw.csv> <title>"""
import collections
import csv
import io
import re
import sys


def _rows(path):
    text = open(path, errors="replace").read()
    start = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("swf::(anonymous namespace)::", "").replace("swf::", "")
    return name.strip()


def launches(path, title):
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in _rows(path):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
        k = short(r["Kernel Name"])
        tot[k] = tot.get(k, 0.0) + ms
        cnt[k] += 1
    total = sum(tot.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)")
    print(f"# total device time {total:.1f} ms over {sum(cnt.values())} launches")
    print(f"{'kernel':<48} {'launches':>8} {'total_ms':>10} {'share':>7} {'ms/launch':>10}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:<48} {cnt[k]:>8} {v:>10.2f} {100 * v / total:>6.2f}% {v / cnt[k]:>10.3f}")


def full(path, title):
    rows = _rows(path)
    want = {
        "gpu__time_duration.sum": "time",
        "sm__cycles_elapsed.avg.per_second": "clk",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu",
        "dram__bytes_read.sum": "dram_r",
        "dram__bytes_write.sum": "dram_w",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "lts__t_sector_hit_rate.pct": "l2hit",
        "launch__registers_per_thread": "regs",
        "launch__grid_size": "grid",
        "launch__block_size": "block",
    }
    if rows and "Metric Name" not in rows[0]:  # wide format: one row per launch, metrics as columns
        print(f"# {title}")
        units = rows[0]
        for r in rows[1:]:
            k = short(r.get("Kernel Name", "?"))
            vals = {}
            for m, key in want.items():
                if m in r:
                    try:
                        vals[key] = float(str(r[m]).replace(",", ""))
                        vals[key + "_u"] = units.get(m, "")
                    except ValueError:
                        pass
            print(k + ": " + ", ".join(f"{key} {vals[key]:g} {vals.get(key + '_u', '')}".strip()
                                       for key in want.values() if key in vals))
        return


if __name__ == "__main__":
    mode, path, title = sys.argv[1], sys.argv[2], sys.argv[3]
    launches(path, title) if mode == "launches" else full(path, title)
