cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY'
import sys, time
sys.path.insert(0,'.')
from paper_1905_11722_b200 import named_graph, Solver
for p in (0.4, 0.3, 0.25, 0.2):
    g=named_graph('random-dag',depth=516,edge_prob=p,seed=0)
    t=time.time(); s=Solver(g,'full'); t1=time.time()
    pl=s.plan(2*g.total_memory); t2=time.time()
    tm=s.timings()
    print(p, 'F', s.dev.size, 'build', round(t1-t,3), 'solve', round(t2-t1,3), 'X', pl.stats.transitions, 't*', pl.objective_value, tm, flush=True)
    pl2=s.plan(2*g.total_memory); t3=time.time(); print(' again', round(t3-t2,3), flush=True)
    s.close()
PY
