#!/bin/bash
# --fmad=false (the product: bit-parity with the oracle) vs --fmad=true A/B:
# both libraries run the same C2 steps, interleaved, and the drift of the
# contracted build against the product build is printed (iterations, relative
# L2 of K and u_next).  Needs build_ab/fmad/lib/libirkdev.so
# (make -C paper_2010_11377_b200 FMAD=true OUT=$PWD/build_ab/fmad/lib OBJ=$PWD/build_ab/fmad/obj).
for round in 1 2 3; do
  unset IRK_LIB; timeout 300 python tools/fmad_step.py gpurun_out/fmad_false_$round.npz 4
  IRK_LIB=$PWD/build_ab/fmad/lib/libirkdev.so timeout 300 python tools/fmad_step.py gpurun_out/fmad_true_$round.npz 4
done
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/fmad_false_1.npz"), np.load("gpurun_out/fmad_true_1.npz")
rl = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
for k in range(4):
    print(f"step {k}: iterations {int(a[f'it{k}'])} vs {int(b[f'it{k}'])}, "
          f"rel K {rl(b[f'K{k}'], a[f'K{k}']):.2e}, rel u_next {rl(b[f'u{k}'], a[f'u{k}']):.2e}")
for tag in ("false", "true"):
    ms = [float(np.load(f"gpurun_out/fmad_{tag}_{r}.npz")[f"ms{k}"]) for r in (1, 2, 3) for k in range(4)]
    print(f"fmad={tag}: median ms/step {np.median(ms):.3f} over {len(ms)} steps")
PY
rm -f gpurun_out/fmad_*.npz  # keep gpurun_out small enough to travel back
