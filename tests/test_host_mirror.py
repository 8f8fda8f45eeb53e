"""Host-side mirror of the reference step API (paper_1803_02977_b200/lem.py):
names, defaults and error behaviour, checked without a GPU."""
import numpy as np
import pytest

import paper_1803_02977_b200 as lem
from paper_1803_02977_b200.lem import strategy_from_string


def test_defaults_match_reference():
    # include/lem/erosion.hpp:16-24, include/lem/config.hpp:23-26
    p = lem.SimParams()
    assert (p.K, p.m_exp, p.n_exp, p.uplift_rate, p.dt, p.epsilon, p.dx, p.dy, p.max_newton_iters) == (
        2e-6, 0.5, 1.0, 2e-3, 1000.0, 1e-6, 1.0, 1.0, 100)
    c = lem.RunConfig()
    assert (c.width, c.height, c.seed, c.timesteps) == (500, 500, 42, 120)


def test_strategy_names():
    assert strategy_from_string("rb_gpu") is lem.StrategyKind.kRbGpu
    assert strategy_from_string("rb_private_queues") is lem.StrategyKind.kRbPrivateQueues
    assert strategy_from_string("nope") is None
    assert len(lem.lem.kAllStrategies) == 7


@pytest.mark.parametrize("kw,msg", [({"dt": 0}, "dt"), ({"K": -1}, "K"), ({"n_exp": 0}, "n_exp"),
                                    ({"max_newton_iters": 0}, "max_newton_iters"), ({"dy": 0}, "spacing")])
def test_params_validate(kw, msg):
    with pytest.raises(lem.ConfigError, match=msg):
        lem.SimParams(**kw).validate()


def test_step_rejects_unsupported_setups():
    g = lem.GridGraph(8, 8)
    e = np.zeros((8, 8))
    ws = lem.SimWorkspace()
    with pytest.raises(lem.ConfigError, match="CPU strategy"):
        lem.strategy_step(e, g, lem.SimParams(), lem.StepSetup(), lem.Strategy(lem.StrategyKind.kRbSerial), ws)
    with pytest.raises(lem.ConfigError, match="mfd_exponent"):  # config.cpp:166
        lem.strategy_step(e, g, lem.SimParams(), lem.StepSetup(routing=lem.Routing.kMfd, mfd_exponent=0.0),
                          lem.Strategy(), ws)
    with pytest.raises(lem.ConfigError, match="mfd_exponent"):
        lem.RunConfig(routing=lem.Routing.kMfd, mfd_exponent=-1.0).validate()
    with pytest.raises(lem.ConfigError, match="queue"):
        lem.strategy_step(e, g, lem.SimParams(), lem.StepSetup(order=lem.OrderKind.kStack), lem.Strategy(), ws)
    with pytest.raises(lem.ConfigError, match="shape"):
        lem.strategy_step(np.zeros((8, 9)), g, lem.SimParams(), lem.StepSetup(), lem.Strategy(), ws)


def test_neighborhood_make():
    assert lem.Neighborhood.make(4).connectivity == 4
    with pytest.raises(lem.ConfigError, match="hexagonal"):
        lem.Neighborhood.make(6)
    with pytest.raises(lem.ConfigError):
        lem.Neighborhood.make(3)


def test_convergence_error_carries_cell():
    e = lem.ConvergenceError(17, "boom")
    assert e.cell() == 17 and isinstance(e, lem.Error)
