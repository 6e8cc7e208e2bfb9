"""First events of a traced host-resident call: what the H2D queue and the compute
streams do during start-up.  python tools/trace_head.py [n] [events] [options-dict]"""
import sys

sys.path.insert(0, ".")
from paper_1510_05041_b200 import RunOptions, build_call, run_call  # noqa: E402
from paper_1510_05041_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nev = int(sys.argv[2]) if len(sys.argv) > 2 else 120
kw = eval(sys.argv[3]) if len(sys.argv) > 3 else {}
call = build_call("gemm", m=n, n=n, k=n, tile_size=1024, seed=0, alpha=1.0, beta=1.0)
eng = get_engine([0], 8)
for x in (call.a, call.b, call.c):
    eng.register_host(x.matrix.storage)
run_call(call, options=RunOptions(**kw))
res = run_call(call, options=RunOptions(record_trace=True, **kw))
tr = sorted(res.trace, key=lambda e: e.time_start)
tasks = {t.task_id: t for t in res.plan.tasks}
print("makespan ms", round(res.metrics.makespan_seconds * 1e3, 2))
for e in tr[:nev]:
    t = tasks.get(e.task_id)
    where = f"C({t.out_ref.i},{t.out_ref.j})" if t is not None else ""
    print(f"{e.event:6s} lane {e.stream:2d} task {e.task_id:4d} {where:9s} k {e.k:3d} "
          f"{e.time_start * 1e3:8.3f} -> {e.time_end * 1e3:8.3f} ms")
