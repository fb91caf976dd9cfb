"""C-ABI boundary checks that need no GPU: the library loads and exports every
function include/tlru.h declares; host-only validation returns the documented codes."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tlru.h")


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2510_15152_b200 import _abi
    return _abi


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:tlru_status|const char\*|uint64_t)\s+(tlru_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("tlru_generate_traces", "tlru_simulate_batch", "tlru_tail_metrics", "tlru_trace_from_turns"):
        assert must in names


def test_library_exports_every_declared_symbol(abi):
    names = declared_functions()
    out = subprocess.check_output(["nm", "-D", "--defined-only", abi.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (tlru_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(abi.EXPORTS) == set(names)
    for n in names:
        getattr(abi.lib, n)


def test_library_is_sm100a(abi):
    out = subprocess.check_output(["cuobjdump", "--list-elf", abi.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_host_validation_codes(abi):
    g = abi.GenParams()
    out = ctypes.c_uint64()
    assert abi.lib.tlru_trace_max_events(ctypes.byref(g), ctypes.byref(out)) == 1  # EINVAL: N == 0
    assert b"num_conversations" in abi.lib.tlru_last_error()
    from paper_2510_15152_b200.inputs import preset
    for k, v in preset("wildchat", 1, 1000).items():
        setattr(g, k, v)
    assert abi.lib.tlru_trace_max_events(ctypes.byref(g), ctypes.byref(out)) == 0
    assert out.value == 1000 * 64 and abi.lib.tlru_last_error() == b""
    g.block_tokens = 0
    assert abi.lib.tlru_trace_max_events(ctypes.byref(g), ctypes.byref(out)) == 1
    assert abi.lib.tlru_set_sim_options(0, 33) == 1
    assert abi.lib.tlru_set_sim_options(40000, 0) == 2
    assert abi.lib.tlru_set_sim_options(0, 0) == 0


def test_pool_and_tail_host_validation(abi):
    """Host-side checks of the pooled-metrics calls (no device work is reached)."""
    fake = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    pool = (ctypes.c_uint32 * 3)(0, 0xFFFFFFFF, 2)
    sz = ctypes.c_size_t()
    assert abi.lib.tlru_pool_workspace_size(3, ctypes.byref(sz)) == 0 and sz.value >= 12
    assert abi.lib.tlru_pool_histograms(fake, 3, 10, pool, 2, fake, fake, sz.value, None) == 1  # pool[2] >= npool
    assert b"pool[2]" in abi.lib.tlru_last_error()
    assert abi.lib.tlru_pool_histograms(None, 3, 10, pool, 3, fake, fake, sz.value, None) == 1  # hist NULL
    assert abi.lib.tlru_pool_histograms(fake, 3, 0, pool, 3, fake, fake, sz.value, None) == 1  # bins == 0
    assert abi.lib.tlru_tail_from_histograms(fake, 2, 70000, None, None, None, 12.5, fake, None) == 1
    assert abi.lib.tlru_tail_from_histograms(fake, 2, 10, None, None, None, -1.0, fake, None) == 1
    assert abi.lib.tlru_tail_from_histograms(None, 0, 10, None, None, None, 1.0, None, None) == 0  # ns == 0


def test_sim_workspace_rejects_unknown_policy(abi):
    tr = (abi.Trace * 1)()
    tr[0].num_events = 0
    inst = (abi.Instance * 1)()
    inst[0].policy = 10  # beyond ETLRU_FORCED: not built
    sz = ctypes.c_size_t()
    assert abi.lib.tlru_sim_workspace_size(tr, 1, inst, 1, ctypes.byref(sz)) == 4  # EUNSUPPORTED
    inst[0].policy = 1
    inst[0].trace = 5
    assert abi.lib.tlru_sim_workspace_size(tr, 1, inst, 1, ctypes.byref(sz)) == 1  # EINVAL
    inst[0].trace = 0
    assert abi.lib.tlru_sim_workspace_size(tr, 1, inst, 1, ctypes.byref(sz)) == 0 and sz.value > 0


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_15152_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f


def _header_struct_fields(name):
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    m = re.search(r"typedef struct\s*\{([^{}]*)\}\s*" + name + r"\s*;", src)
    assert m, name
    fields = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        ty, names = decl.split(None, 1) if not decl.startswith("const") else decl.split(None, 2)[1:]
        for n in names.split(","):
            fields.append(n.strip().lstrip("*"))
    return fields


@pytest.mark.parametrize("cname,pyname", [("tlru_gen_params", "GenParams"), ("tlru_trace", "Trace"),
                                          ("tlru_instance", "Instance"), ("tlru_sim_stats", "SimStats")])
def test_ctypes_structs_mirror_the_header(abi, cname, pyname):
    assert [f for f, _ in getattr(abi, pyname)._fields_] == _header_struct_fields(cname)


@pytest.mark.parametrize("cname,dt", [("tlru_result", "RESULT_DTYPE"), ("tlru_tail", "TAIL_DTYPE")])
def test_numpy_dtypes_mirror_the_header(abi, cname, dt):
    assert list(getattr(abi, dt).names) == _header_struct_fields(cname)
