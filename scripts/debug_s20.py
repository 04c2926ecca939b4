import faulthandler, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(100, exit=True)
import paper_2403_05802_b200 as sfg
ctx = sfg.Context(0)
for sc in (18, 19, 20, 21, 20, 22):
    g = ctx.gen_rmat(7, sc, 16 << sc)
    ctx.synchronize()
    print("gen", sc, g.view().nvals, flush=True)
    for fmt in (("CSR", "DCSR", "ELL", "HYB(8)") if sc < 19 else ("CSR", "DCSR", "HYB(8)", "HYB(1)", "HYB(100)")):
        h = ctx.convert(g, fmt)
        ctx.synchronize()
        print("  ", fmt, "ok", flush=True)
print("ALL OK")
