"""profiles/bench_kernel_ncu.json from two ncu captures of the bench workload:
  launches: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
            -k regex:wave_walk --csv --log-file <launches.csv> python bench.py --steps 1 ...
  full:     ncu --set full -k regex:wave_walk -s N -c 1 -o <full> python bench.py ...
usage: python tools/walk_profile.py launches.csv full.ncu-rep projections out.json"""
import csv
import io
import json
import subprocess
import sys

launches, full, n_proj, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]

# 1. per-launch DRAM bytes and durations of every walk launch
tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
n_launch = set()
hdr = None
for r in csv.reader(open(launches)):
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    m = d.get("Metric Name")
    if m in tot and "wave_walk" in d.get("Kernel Name", ""):
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6,
                 "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1.0)
        tot[m] += v * scale
        n_launch.add(d["ID"])

# 2. one launch under --set full: instructions, warp iterations (the loop-top vote), issue
raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
num = lambda k: float(d[k].replace(",", ""))  # noqa: E731
inst = num("smsp__inst_executed.sum")
sass = subprocess.run(["ncu", "-i", full, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(sass)))
h = srows[1]
ie, src = h.index("Instructions Executed"), h.index("Source")
votes = [int(r[ie]) for r in srows[2:] if len(r) > ie and "VOTE.ANY" in r[src] and r[ie].isdigit()]
# a loop trip (one loop-top vote) is XSW_INNER = 3 block steps (wavefront.cu): per warp step slot
steps_per_trip = 3
warp_it = max(votes) * steps_per_trip
res = {
    "kernel": d.get("Kernel Name", "wave_walk")[:120],
    "source": "tools/profile_round.sh: ncu launch metrics over every walk launch of the bench run, and one "
              "--set full launch (instructions per warp step slot = sm instructions / (executions of the "
              "loop-top VOTE.ANY x 3 steps per trip))",
    "walk_launches_per_projection": len(n_launch) / n_proj,
    "walk_dram_bytes_read_per_projection": tot["dram__bytes_read.sum"] / n_proj,
    "walk_dram_bytes_write_per_projection": tot["dram__bytes_write.sum"] / n_proj,
    "walk_dram_bytes_per_projection": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / n_proj,
    "walk_time_ms_per_projection_under_ncu": tot["gpu__time_duration.sum"] / n_proj,
    "walk_warp_instructions_per_warp_iteration": inst / warp_it,
    "walk_steps_per_loop_trip": steps_per_trip,
    "walk_issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "walk_warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "walk_l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "walk_registers": num("launch__registers_per_thread"),
    "full_capture_duration_ms": num("gpu__time_duration.sum") * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
                                                                  "usecond": 1e-3}.get(rows[1][rows[0].index("gpu__time_duration.sum")], 1.0),
    "full_capture_dram_read_bytes": num("dram__bytes_read.sum") * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
        rows[1][rows[0].index("dram__bytes_read.sum")], 1.0),
}
# walker state read by the walk per ray: t, texit, target, tn x3, dt x3, rd x3, 4 mu (fp64),
# 3 voxel indices (i32), flags (u8) = 141 B; rays per projection from the bench line if given
if len(sys.argv) > 5:
    rays = float(sys.argv[5])
    res["walker_state_bytes_per_ray"] = 141
    res["walker_state_dram_share"] = min(1.0, 141.0 * rays / max(1.0, res["walk_dram_bytes_read_per_projection"]))
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
