"""The reference's own test modules, run unchanged against this package.

The files next to this one (helpers.py, test_analytics.py, test_traffic.py,
test_acceptance.py, test_partitioning.py, test_cli.py) are verbatim copies of
/root/reference/pkg/tests -- TEST INFRASTRUCTURE, kept byte-identical so the
reference's acceptance criteria judge the drop-in (VERDICT r01 "Next" 8). This
conftest (written here, not copied) makes ``import netmeter`` resolve to
``paper_2510_14050_b200`` and supplies the scheduler fixtures of the
reference's conftest.py. Everything except test_partitioning.py calls the
device path, so those modules carry the ``gpu`` marker.

Deselected, with the reason (SURVEY.md 2 / DESIGN.md 6 scope):
* test_acceptance.py::test_senders_laws -- the P2300 senders algebra
  (senders.py) is host-side emulation with no device counterpart;
* test_acceptance.py::test_scaling_smoke_r4_vs_r1 -- asserts that the host
  thread pool speeds up one matrix's reductions 1.25x from 1 to 4 workers; on
  the device that reduction is one kernel and a group spreads *windows*
  (tests/test_gpu_group.py covers the group).
"""

import sys
import types

import pytest

import paper_2510_14050_b200 as _pkg
from paper_2510_14050_b200 import analytics, bench, cli, partitioning, resources, traffic

sys.modules.setdefault("netmeter", _pkg)
for _name, _mod in (("analytics", analytics), ("traffic", traffic), ("resources", resources),
                    ("partitioning", partitioning), ("bench", bench), ("cli", cli)):
    sys.modules.setdefault(f"netmeter.{_name}", _mod)
if "netmeter.senders" not in sys.modules:  # imported at the top of test_acceptance.py only
    _senders = types.ModuleType("netmeter.senders")

    def _out_of_scope(*a, **k):
        raise NotImplementedError("senders algebra is out of scope (DESIGN.md 6)")

    for _n in ("bulk", "exec_on", "just", "sync_wait", "then"):
        setattr(_senders, _n, _out_of_scope)
    sys.modules["netmeter.senders"] = _senders

_DESELECT = {"test_senders_laws", "test_scaling_smoke_r4_vs_r1"}


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        if "reference_suite" not in str(it.fspath):
            keep.append(it)
            continue
        if it.originalname in _DESELECT or it.name in _DESELECT:
            drop.append(it)
            continue
        if not str(it.fspath).endswith("test_partitioning.py"):
            it.add_marker(pytest.mark.gpu)
        keep.append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep


@pytest.fixture
def inline_sched():
    return resources.make_inline_scheduler()


@pytest.fixture
def pool_sched():
    with resources.make_pool_scheduler(4) as sched:
        yield sched


@pytest.fixture
def group_sched():
    with resources.make_group_scheduler([2, 2, 2, 2]) as sched:
        yield sched


@pytest.fixture(params=["inline", "pool", "group"])
def any_sched(request):
    if request.param == "inline":
        yield resources.make_inline_scheduler()
    elif request.param == "pool":
        with resources.make_pool_scheduler(4) as sched:
            yield sched
    else:
        with resources.make_group_scheduler([2, 2, 2, 2]) as sched:
            yield sched
