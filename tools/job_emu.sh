# FP64 emulation on int8 tensor cores: accuracy tests, builds with it on/off, bench lines.
set -u
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
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rA -k "emulated or two_contexts" > gpurun_out/pytest_emu.log 2>&1; tail -8 gpurun_out/pytest_emu.log
timeout 900 python - <<'PY' > gpurun_out/emu_build.txt 2>&1
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1307_2665_b200 as P
from paper_1307_2665_b200 import solver, problems, _native
for cfg, L in ((2, 6), (3, 7), (5, 8)):
    tree, nodes = P.build_tree(P.Rectangle(0, 1, 0, 1), L, 16)
    inp = solver.prepare(tree, nodes, problems.coefficients(cfg))
    out = {}
    for sl in (0, 8, 7):
        _native.context().set("emu_slices", sl)
        st = solver.build_device(inp)
        assert not solver.check_build(st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            st = solver.build_device(inp)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        out[sl] = (st.root_T.device_tensor.clone(), dt)
    _native.context().set("emu_slices", 0)
    T0 = out[0][0]
    for sl in (8, 7):
        d = float((out[sl][0] - T0).abs().max() / T0.abs().max())
        print(f"cfg{cfg} L{L}: slices {sl}: root T vs DMMA {d:.2e}; build {out[sl][1]*1e3:.1f} ms vs DMMA {out[0][1]*1e3:.1f} ms", flush=True)
PY
cat gpurun_out/emu_build.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_emu.csv python /tmp/one_emu.py > gpurun_out/ncu_emu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_emu.csv 2>/dev/null | head -16
