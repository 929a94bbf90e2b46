"""Print the stall-reason breakdown (pc sampling) and pipe utilisation of an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:60]
    print("==", name, "dur", r[h.index("gpu__time_duration.sum")])
    for w in ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active"]:
        if w in h:
            print(f"   {w}: {r[h.index(w)]}")
    st = []
    for i, w in enumerate(h):
        if w.startswith("smsp__pcsamp_warps_issue_stalled_") and not w.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), w.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{w} {v / tot * 100:.1f}%" for v, w in sorted(st, reverse=True)[:8]))
