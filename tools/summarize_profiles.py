"""Turn the raw ncu outputs of tools/profile_round.sh into committed summaries:
profiles/<tag>_kernel_shares.txt  (launch list: per-kernel share of a frame)
profiles/<tag>_ncu_top.txt        (full-set metrics + stall mix per kernel)
profiles/ncu_traffic.json         (DRAM bytes per launch, read by bench.py)"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAUNCH_CMD = os.environ.get("LAUNCH_CMD", "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs (C2)")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows[hdr_i + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("vp::", "")
            agg[name][0] += float(r[vi].replace(",", ""))
            agg[name][1] += 1
    return agg


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("vp::", "")

        def g(k):
            return (float(r[hdr.index(k)].replace(",", "")), units[hdr.index(k)]) if k in hdr else (None, "")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        out[name] = dict(
            time=g("gpu__time_duration.sum"), dram_read=g("dram__bytes_read.sum"),
            dram_write=g("dram__bytes_write.sum"),
            sm_pct=g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            mem_pct=g("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
            warps_active=g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            regs=g("launch__registers_per_thread"), stalls=st[:5],
            inst=g("smsp__inst_executed.sum"), red=g("lts__t_sectors_srcunit_tex_op_red.sum"),
            atom=g("lts__t_sectors_srcunit_tex_op_atom.sum"),
            atom_unit=g("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"), l1_red=g("l1tex__t_requests_pipe_lsu_mem_global_op_red.sum"),
            l1_atom=g("l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum"),
            pipes={k: g(m)[0] for k, m in PIPES.items()})
    return out


# what limits a kernel that is not bandwidth-bound: issue slots and pipe utilisation
PIPES = {"issue": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
         "alu": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
         "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
         "lsu": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "l2": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
         "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"}


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def main(tag):
    src = os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    agg = launches(os.path.join(src, f"{tag}_launches.csv"))
    tot = sum(v[0] for v in agg.values())
    with open(os.path.join(dst, f"{tag}_kernel_shares.txt"), "w") as f:
        f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none, serialised, cold): "
                f"{LAUNCH_CMD}; {sum(v[1] for v in agg.values())} launches\n")
        f.write(f"{'kernel':28s} {'launches':>8s} {'total_us':>10s} {'us/launch':>10s} {'share':>7s}\n")
        for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
            f.write(f"{k:28s} {n:8d} {t / 1e3:10.1f} {t / 1e3 / n:10.2f} {100 * t / tot:6.1f}%\n")
    fl = full(os.path.join(src, f"{tag}_top.ncu-rep"))
    traffic, pipes, inst, atomics = {}, {}, {}, {}
    with open(os.path.join(dst, f"{tag}_ncu_top.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none, one launch per kernel (C2 frame ~10)\n")
        for k, d in fl.items():
            rb = to_bytes(*d["dram_read"]) if d["dram_read"][0] is not None else 0
            wb = to_bytes(*d["dram_write"]) if d["dram_write"][0] is not None else 0
            traffic[k] = rb + wb
            f.write(f"== {k}\n")
            f.write(f"   duration {d['time'][0]} {d['time'][1]}; DRAM read {rb / 1e6:.3f} MB, write {wb / 1e6:.3f} MB\n")
            f.write(f"   SM throughput {d['sm_pct'][0]:.1f}%, memory throughput {d['mem_pct'][0]:.1f}%, "
                    f"warps active {d['warps_active'][0]:.1f}%, {int(d['regs'][0])} regs/thread\n")
            f.write("   stalls per issue: " + ", ".join(f"{n}={v:.2f}" for v, n in d["stalls"]) + "\n")
            pipes[k] = {n: round(v, 1) for n, v in d["pipes"].items() if v is not None}
            f.write("   utilisation %: " + ", ".join(f"{n} {v}" for n, v in pipes[k].items()) + "\n")
            us = d["time"][0] * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["time"][1], 1.0)
            if d["inst"][0] is not None:
                inst[k] = d["inst"][0]
                f.write(f"   warp instructions {d['inst'][0]:.0f} ({d['inst'][0] / us / 1e3:.1f} G/s)\n")
            a = {n: d[n][0] for n in ("red", "atom", "l1_red", "l1_atom") if d[n][0] is not None}
            if a:
                atomics[k] = {"l2_red_sectors": a.get("red"), "l2_atom_sectors": a.get("atom"),
                              "l1_red_requests": a.get("l1_red"), "l1_atom_requests": a.get("l1_atom"),
                              "l2_red_atom_sectors_per_s": round(((a.get("red") or 0) + (a.get("atom") or 0))
                                                                 / (us * 1e-6), 1),
                              "l2_atomic_unit_pct": d["atom_unit"][0]}
                f.write("   atomics: L2 RED sectors %s, L2 ATOM sectors %s, L1 RED req %s, L1 ATOM req %s "
                        "(L2 RED+ATOM %.2f G sectors/s; L2 atomic unit busy %s%% of peak)\n"
                        % (a.get("red"), a.get("atom"), a.get("l1_red"), a.get("l1_atom"),
                           atomics[k]["l2_red_atom_sectors_per_s"] / 1e9, d["atom_unit"][0]))
    json.dump({"source": f"profiles/{tag}_ncu_top.txt", "dram_bytes_per_launch": traffic,
               "utilisation_pct": pipes, "warp_inst_per_launch": inst, "atomics_per_launch": atomics},
              open(os.path.join(dst, "ncu_traffic.json"), "w"), indent=1)
    print(open(os.path.join(dst, f"{tag}_kernel_shares.txt")).read())
    print(open(os.path.join(dst, f"{tag}_ncu_top.txt")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
