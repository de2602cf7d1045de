set -u
mkdir -p gpurun_out
cat > /tmp/one_emu.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), 8, 16)
inp = solver.prepare(tree, nodes, problems.coefficients(5))
_native.context().set("emu_slices", 8)
st = solver.build_device(inp); torch.cuda.synchronize()
st = solver.build_device(inp); torch.cuda.synchronize()
print("ok")
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_emu.csv python /tmp/one_emu.py > gpurun_out/ncu_emu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_emu.csv 2>/dev/null | head -25
