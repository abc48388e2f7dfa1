"""Turn a round's gpurun_out/ evidence (tools/round_profiles.sh) into profiles/<round>_* files
(dev tool, runs without a GPU).  usage: round_summaries.py r02"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summarise  # noqa: E402

rnd = sys.argv[1]
G, P = Path("gpurun_out"), Path(sys.argv[2] if len(sys.argv) > 2 else "profiles")
P.mkdir(parents=True, exist_ok=True)


def val(k, name):
    v = k.get(name)
    return None if v is None else float(v[0])


def to_bytes(k, name):
    v = k.get(name)
    if v is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(v[1], 1)
    return float(v[0]) * scale


def dump(name, obj):
    (P / f"{rnd}_{name}").write_text(json.dumps(obj, indent=1))
    print(P / f"{rnd}_{name}")


cmds = {
    "summary_1024": "ncu --set full -k regex:k_brick_summary -s 2 -c 1 python bench.py --steps 2 "
                    "--warmup 3 --no-cpu --frame-only (cold rebuild engine, 1024^3)",
    "frame_1024": "ncu --set full -k regex:'k_segments_brick|k_integrate_segments|k_flags_tiles|"
                  "k_tree_chunk|k_leaves_coop|k_presence' -s 12 -c 8 python bench.py --steps 2 "
                  "--warmup 3 --no-cpu --frame-only (interactive frame: warm rebuild + render)",
    "kd_1024": "ncu --set full -k regex:'k_classify_pack|k_levels' -c 3 python tools/prof_kd.py "
               "1024 hybrid 0.6 1",
    "multi_1024": "ncu --set full -k regex:k_integrate_multi -c 1 python bench.py --channels 4 "
                  "--steps 1 --warmup 3 --no-cpu",
}
for rep, note in cmds.items():
    f = G / f"{rep}.ncu-rep"
    if f.exists():
        dump(f"ncu_{rep}.json", {"report": str(f), "command": note, "kernels": summarise(str(f))})

# k_brick_summary traffic per launch (bench.py roofline.traffic)
f = G / "summary_1024.ncu-rep"
if f.exists():
    k = summarise(str(f))[0]
    rd, wr = to_bytes(k, "dram__bytes_read.sum"), to_bytes(k, "dram__bytes_write.sum")
    dump("ncu_k_brick_summary.json", {
        "kernel": k["kernel"], "command": cmds["summary_1024"], "dram_bytes_read": rd,
        "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": 1024 ** 3 + 4 * 128 ** 3,
        "duration_us": val(k, "gpu__time_duration.sum")})

# render views: L1 hit rate per TF (bench.py render_by_t.l1_hit_pct_ncu)
for t in ("0.6", "0.3", "0.0"):
    f = G / f"render_t{t}.ncu-rep"
    if not f.exists():
        continue
    ks = summarise(str(f))
    integ = [k for k in ks if "integrate" in k["kernel"]]
    seg = [k for k in ks if "segments" in k["kernel"]]
    dump(f"ncu_render_t{t.replace('.', '')[:2]}.json", {
        "command": f"ncu --set full -k regex:'k_segments_brick|k_integrate_segments' -s 2 -c 2 "
                   f"python tools/prof_render.py 1024 lbvh {t} 32 (1920x1080, az 30 el 15)",
        "l1_hit_pct": val(integ[0], "l1tex__t_sector_hit_rate.pct") if integ else None,
        "l1_hit_pct_segments": val(seg[0], "l1tex__t_sector_hit_rate.pct") if seg else None,
        "kernels": ks})

for src, dst in (("bench.json", "bench_interactive_1024.json"),
                 ("bench_ref.json", "bench_reference_arm.json"),
                 ("bench_mc4.json", "bench_multichannel4_1024.json"),
                 ("configs.json", "configs.json"),
                 ("launches_interactive_frame.csv", "launches_interactive_frame.csv"),
                 ("launches_mc4.csv", "launches_multichannel4_frame.csv"),
                 ("launches_hybrid_1024.csv", "launches_hybrid_rebuild_1024.csv"),
                 ("launches_kd_deep_512.csv", "launches_kd_deep_mls32_512.csv"),
                 ("smoke.log", "smoke.log")):
    if (G / src).exists():
        shutil.copy(G / src, P / f"{rnd}_{dst}")
if (G / "pytest_gpu.log").exists():
    tail = (G / "pytest_gpu.log").read_text().splitlines()[-3:]
    (P / f"{rnd}_pytest_gpu_tail.txt").write_text("\n".join(tail) + "\n")
for csv in sorted(P.glob(f"{rnd}_launches_*.csv")):
    out = subprocess.run([sys.executable, "tools/launch_summary.py", str(csv)],
                         capture_output=True, text=True).stdout
    csv.with_suffix(".txt").write_text(out)
