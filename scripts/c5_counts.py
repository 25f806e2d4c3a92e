import sys; sys.path.insert(0, '.')
import paper_2401_09961_b200 as pu
xs = [pu.config_scene("c5", b)[1] for b in range(64)]
res = pu.unwrap_many(xs, dtype="fp64", concurrency=8)
print("C5 fp64 outer", sum(len(r.trace.records) for r in res), "pcg", sum(sum(q.cg_iters for q in r.trace.records) for r in res))
print("img0", len(res[0].trace.records), sum(q.cg_iters for q in res[0].trace.records))
