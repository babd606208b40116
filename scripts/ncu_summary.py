"""Summarise a profiling pass (scripts/profile_round.sh output) into profiles/.

usage: python scripts/ncu_summary.py gpurun_out/<tag> <round-name> [dest]
writes profiles/<round>_<name>_launches.csv (kernel, duration ns), profiles/<round>_<name>_full.txt
(key metrics of the `ncu --set full` capture) and merges profiles/traffic.json.  <name> is a config
(c2 ...) or a config variant (c2_csr, c2_R8: the config through CSR / at 8 vectors per GPU); the
profiling script writes specs.json mapping each name to its R per GPU."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out


def num(v):
    return float(v.replace(",", ""))


def main(src, rnd, dest=None):
    prof = dest or os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    tpath = os.path.join(prof, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    specs = {}
    sp = os.path.join(src, "specs.json")
    if os.path.exists(sp):
        specs = json.load(open(sp))
    for c in (list(specs) or ["c1", "c2", "c3", "c4", "c5", "pd"]):
        ll = os.path.join(src, f"launchlist_{c}.csv")
        if os.path.exists(ll):
            rows = read_ncu_csv(ll)
            per = collections.defaultdict(list)
            with open(os.path.join(prof, f"{rnd}_{c}_launches.csv"), "w") as f:
                f.write("id,kernel,grid,block,duration_ns\n")
                for d in rows:
                    if d["Metric Name"] != "gpu__time_duration.sum":
                        continue
                    k = d["Kernel Name"].split("(")[0]
                    per[k].append(num(d["Metric Value"]))
                    f.write(f'{d["ID"]},"{d["Kernel Name"][:90]}",{d["Grid Size"]},{d["Block Size"]},{d["Metric Value"]}\n')
            tot = sum(sum(v) for v in per.values())
            with open(os.path.join(prof, f"{rnd}_{c}_launches_summary.txt"), "w") as f:
                f.write(f"# {c}: launch list of one bench step (ncu gpu__time_duration.sum, clock-control none;\n"
                        "# cold-cache serialised replays: compare shares, not absolutes)\n")
                for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                    f.write(f"{k:60s} launches={len(v):5d} total_ms={sum(v) / 1e6:9.3f} "
                            f"mean_us={sum(v) / len(v) / 1e3:9.2f} share={sum(v) / tot:6.3f}\n")
        dr = os.path.join(src, f"dram_{c}.csv")
        if os.path.exists(dr):
            rows = read_ncu_csv(dr)
            agg = collections.defaultdict(list)
            name = None
            for d in rows:
                agg[d["Metric Name"]].append(num(d["Metric Value"]))
                name = d["Kernel Name"]
            n = len(agg["gpu__time_duration.sum"])
            rd = sum(agg["dram__bytes_read.sum"]) / n
            wr = sum(agg["dram__bytes_write.sum"]) / n
            t = sum(agg["gpu__time_duration.sum"]) / n
            traffic[c] = {"tma": int("tma" in (name or "")), "kernel": (name or "")[:160], "launches": n,
                          "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
                          "mean_duration_ns": t, "round": rnd, "R_loc": specs.get(c, {}).get("R_loc"),
                          "note": "mean over steady-state step launches (ncu dram__bytes_read.sum + "
                                  "dram__bytes_write.sum)"}
        rep = os.path.join(src, f"full_{c}.ncu-rep")
        if os.path.exists(rep):
            out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                                 text=True).stdout
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            with open(os.path.join(prof, f"{rnd}_{c}_full.txt"), "w") as f:
                f.write(f"# {c}: ncu --set full --clock-control none, one step-kernel launch\n")
                for d in csv.DictReader(io.StringIO(out)):
                    f.write(f'{d["Section Name"][:34]:34s} {d["Metric Name"][:52]:52s} {d["Metric Value"]} '
                            f'{d["Metric Unit"]}\n')
                rr = list(csv.reader(io.StringIO(raw)))
                if len(rr) >= 3:
                    keys = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                            "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
                            "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
                    f.write("# raw counters\n")
                    for k, u, v in zip(rr[0], rr[1], rr[2]):
                        if k in keys:
                            f.write(f"{k} = {v} {u}\n")
                    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v) for k, v in zip(rr[0], rr[2])
                          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
                    st = sorted(((k, num(v)) for k, v in st if v.replace(",", "").replace(".", "").isdigit()),
                                key=lambda kv: -kv[1])
                    tot = sum(v for _, v in st) or 1.0
                    f.write("# warp stall samples (share)\n")
                    for k, v in st[:10]:
                        f.write(f"stall {k:28s} {v / tot:6.3f}\n")
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
