"""pytest plugin: run the REFERENCE's own test suite with gpu0 as the
default device (harness, not a test module).

    python scripts/run_reference_suite.py [--fake]

Registers tidepool_plugin into the unmodified reference, makes gpu0 the
default device (tensors.set_default_device, tensors.py:29-30) and lets
`from_nested` build on the default device too (the reference hard-codes
cpu there, tensors.py:237), so every test that does not name a device runs
its tensors through the B200 table.  TPG_REFSUITE_FAKE=1 swaps the native
library for the CPU test double (tests/fake_native.py).
"""

import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import ref_loader  # noqa: E402

_ref = ref_loader.reference_dir()
if _ref is not None:
    sys.path.insert(0, str(_ref.parent))

import tidepool  # noqa: E402
from tidepool import tensors  # noqa: E402

from paper_1810_08723_b200 import tidepool_plugin  # noqa: E402

_lib = None
if os.environ.get("TPG_REFSUITE_FAKE") == "1":
    from fake_native import FakeNative
    from oracle import oracle
    _lib = FakeNative(oracle.lib())
GPU = tidepool_plugin.register(tidepool, count=1, lib=_lib)[0]
tensors.set_default_device(GPU)

_orig_nested = tensors.tensor_from_nested


def _from_nested(data, dtype=None, device=None):
    return _orig_nested(data, dtype, device or tensors.default_device())


tensors.tensor_from_nested = _from_nested
tidepool.tensor_from_nested = tidepool.from_nested = _from_nested


def pytest_report_header(config):
    return f"tidepool reference from {_ref}; default device {GPU.name} " \
           f"({'fake native' if _lib is not None else 'libtidepool_gpu.so'})"


def pytest_runtest_teardown(item, nextitem):
    """The reference conftest restores the registry only when it does not
    hold exactly 3 devices (cpu + 2 emu); with gpu0 appended, restore the
    2-emulated-device layout the reference tests assume."""
    from tidepool import devices
    if sum(d.type.name == "emu" for d in devices.list_devices()) != 2:
        devices.configure(2)


# Reference tests whose assertions name the default device's identity rather
# than results: they check the registry layout (cpu + 2 emu, no other type),
# call counters / overrides of the *cpu* table, `ensure(t, device=cpu)`
# returning the same handle, shallow (host-memory) exports, or render text
# containing "cpu".  With gpu0 as the default device they fail by
# construction; every other reference test must pass.
ASSUMES_CPU_DEFAULT = {
    "test_acceptance.py::TestAcceptance::test_dispatch_criteria": "counts cpu-table calls",
    "test_acceptance.py::TestAcceptance::test_strict_mode": "ensure(..., cpu) identity",
    "test_cli.py::TestStrictFlag::test_strict_uniform_qr_passes": "cli mixes cpu tensors with default-device tensors under --strict",
    "test_devices.py::TestRegistry::test_default_layout": "registry layout",
    "test_devices.py::TestRegistry::test_configure_zero_emulated": "registry layout",
    "test_devices.py::TestRegistry::test_configure_four_emulated": "registry layout",
    "test_devices.py::TestRegistry::test_env_variable_drives_default": "registry layout",
    "test_devices.py::TestRegistry::test_lookup_by_name": "asserts gpu0 does not exist",
    "test_devices.py::TestBufferConfig::test_cache_disabled_allocates_every_time": "counts cpu allocations",
    "test_dispatch.py::TestOverride::test_counter_counts_dispatches": "counts cpu-table calls",
    "test_dispatch.py::TestOverride::test_wrapper_sees_original_and_restores": "overrides the cpu table",
    "test_dispatch.py::TestOverride::test_fault_injection_propagates": "overrides the cpu table",
    "test_dispatch.py::TestEveryOpDispatches::test_exercising_the_api_bumps_every_table_counter": "counts cpu-table calls",
    "test_interop.py::TestExternalTypes::test_builtin_blob_round_trip": "shallow export needs host memory",
    "test_interop.py::TestExternalTypes::test_foreign_operand_auto_imports": "shallow export needs host memory",
    "test_interop.py::TestExternalTypes::test_foreign_transparency_matches_imported": "shallow export needs host memory",
    "test_ops.py::TestCopyEnsureCast::test_ensure_returns_same_handle_when_matching": "ensure(..., cpu) identity",
    "test_tensors.py::TestRender::test_two_by_three": "render text names the device",
}


def pytest_collection_modifyitems(config, items):
    import pytest
    for item in items:
        key = item.nodeid.split("/")[-1]
        if key in ASSUMES_CPU_DEFAULT:
            item.add_marker(pytest.mark.xfail(reason="assumes cpu default: "
                                              + ASSUMES_CPU_DEFAULT[key], strict=False))
