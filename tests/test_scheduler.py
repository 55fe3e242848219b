"""Scheduling policies (reference scheduler.py:27-105) and the chunked
least-first policy with the paper's task scores:
every schedule partitions the task indices; least-first balances estimated
work on a power-law graph where even splitting does not."""
import numpy as np
import pytest

import graphs as G
from paper_2112_09761_b200 import graph as GR
from paper_2112_09761_b200 import scheduler as S
from paper_2112_09761_b200.executor import VertexTasks


def _pl():
    g = GR.from_edges(G.powerlaw_edges(20000, 4, 3), num_vertices=20000)
    return g, GR.EdgeTaskList(GR.all_edge_tasks(g), reduced=False)


@pytest.mark.parametrize("policy", [S.POLICY_EVEN, S.POLICY_RR, S.POLICY_CHUNKED, S.POLICY_LEAST])
@pytest.mark.parametrize("n", [1, 3, 8])
def test_every_policy_partitions(policy, n):
    g, tasks = _pl()
    sch = S.make_schedule(tasks, n, policy, workers_y=16, graph=g)
    sch.validate_partition(len(tasks))
    assert sch.num_devices == n


def test_least_first_balances_estimated_work():
    g, tasks = _pl()
    w = S.estimated_work(g, tasks, "degree_sum")

    def imb(q):
        loads = [int(w[x].sum()) for x in q]
        return max(loads) / (sum(loads) / len(loads))

    even = S.split_even(tasks, 4)
    lf = S.make_schedule(tasks, 4, S.POLICY_LEAST, workers_y=64, graph=g)
    assert lf.estimated == [int(w[q].sum()) for q in lf.queues]
    assert imb(lf.queues) < 1.01
    assert imb(even.queues) / imb(lf.queues) >= 1.5


def test_least_first_unit_score_is_balanced_counts():
    g, tasks = _pl()
    sch = S.make_schedule(tasks, 4, S.POLICY_LEAST, workers_y=8, graph=g, score="unit")
    sizes = [len(q) for q in sch.queues]
    assert max(sizes) - min(sizes) <= 16


def test_estimator_scores_and_errors():
    g, tasks = _pl()
    e = tasks.edges
    deg = g.degrees.astype(np.int64)
    assert np.array_equal(S.estimated_work(g, tasks, "degree_min"), np.minimum(deg[e[:, 0]], deg[e[:, 1]]))
    assert np.array_equal(S.estimated_work(g, VertexTasks(g.num_vertices), "degree_sum"), deg)
    with pytest.raises(ValueError, match="score"):
        S.estimated_work(g, tasks, "bogus")
    with pytest.raises(ValueError, match="graph"):
        S.make_schedule(tasks, 2, S.POLICY_LEAST)
    with pytest.raises(ValueError):
        S.split_chunked_least_first(np.ones(4, dtype=np.int64), 2, 0)
