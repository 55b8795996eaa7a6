"""Shared-memory wavefronts per rotation of each kernel, from a committed ncu --set full summary
(profiles/r2/ncu_summary_*.md: one 16-rotation launch per kernel) -> profiles/r2/ncu_smem.json.
bench.py divides them by the live launch time for the roofline's smem_view (the L1/shared
crossbar moves one 128-byte wavefront per SM per cycle, B300_MICROARCH.md "LDS/STS")."""
import json
import re
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "profiles/r2/ncu_summary_j.md"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/r2/ncu_smem.json"
rot = 16
out, cur = {}, None
for line in open(src):
    m = re.match(r"## `([A-Za-z_0-9]+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"- (l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum|l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum|"
                 r"gpu__time_duration\.sum): ([0-9.]+)", line)
    if cur and m and cur not in ("keys_init_kernel", "keys_finalize_kernel", "rot_prep_kernel"):
        key = {"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "wavefronts_per_rotation",
               "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_conflicts_per_rotation",
               "gpu__time_duration.sum": "ncu_ms_per_launch"}[m.group(1)]
        v = float(m.group(2))
        out.setdefault(cur, {})[key] = v if key == "ncu_ms_per_launch" else v / rot
json.dump({"per_kernel": out, "rotations_per_launch": rot, "source": src}, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
