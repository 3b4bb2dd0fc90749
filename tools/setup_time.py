"""Host vs device AMG setup wall time for one C2/C3 diagonal block."""
import sys, time
sys.path.insert(0, ".")
import paper_2010_11377_b200 as P

for cells in [int(c) for c in (sys.argv[1:] or ["1024"])]:
    pr = P.make_heat_setup(cells)
    B = P.CsrMatrix(pr.M.row_ptr, pr.M.col_idx, 1.0 * pr.M.vals + 2e-4 * pr.F.vals, pr.M.n_cols)
    P.amg_setup_device(B)  # context / first-touch warm-up
    t = time.perf_counter(); hd = P.amg_setup_device(B); td = time.perf_counter() - t
    t = time.perf_counter(); hh = P.amg_setup(B); th = time.perf_counter() - t
    print(f"cells={cells} n={B.n_rows} levels={hd.sizes()} host {th:.3f} s  device {td:.3f} s  "
          f"same_sizes={hd.sizes() == hh.sizes()}")

# whole solver construction (hierarchies + format conversion + upload), C2
pr = P.make_heat_setup(1024)
t3 = P.make_radau_iia(3)
pc = P.precond_coeff(t3, P.CoeffKind.LowerFactor)
for rep in range(2):
    t = time.perf_counter()
    Pc = P.BlockPreconditioner(pr.M, pr.F, pc, 1e-3, table=t3)
    _ = Pc._dev
    print(f"C2 solver construction {time.perf_counter() - t:.3f} s (setup_seconds {Pc.setup_seconds():.3f})")
    del Pc, _
