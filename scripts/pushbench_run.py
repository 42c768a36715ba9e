"""Run the GPU Push_WL / Push_NoWL pair at europe_osm scale (n = 50,912,018,
batch 1000) and print TTI summary + crossovers."""
import io
import sys

sys.path.insert(0, ".")
from paper_1912_01478_b200.pushbench import BenchConfig, detect_crossovers, run_push_bench, write_tti_csv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_912_018
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S = {}
for v in ("push_wl", "push_nowl"):
    s = run_push_bench(n, BenchConfig(variant=v, repetitions=reps))
    S[v] = s
    m = s.micros()
    q = [0, len(m) // 4, len(m) // 2, 3 * len(m) // 4, len(m) - 1]
    print(v, len(m), "iterations; TTI us at", q, ":", [round(float(m[i]), 1) for i in q],
          "total ms", round(float(m.sum()) / 1e3, 1))
x = detect_crossovers(S["push_wl"], S["push_nowl"])
print("crossovers:", len(x), "first:", x[:5])
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        write_tti_csv(f, [S["push_wl"], S["push_nowl"]])
