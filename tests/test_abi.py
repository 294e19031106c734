"""C-ABI checks that need no GPU: the library loads, exports every symbol include/*.h
declares, host-only helpers work, and device calls fail loudly (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import paper_1811_10573_b200.cppp as cp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    inc = os.path.join(ROOT, "include")
    src = "\n".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc)) if f.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[ \t]*(?:const[ \t]+)?[a-z_0-9]+(?:[ \t]+|[ \t]*\*[ \t]*)([a-z_0-9]+)[ \t]*\(",
                       src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for want in ["cp_init", "mttkrp_dt", "pp_build_operators", "pp_update", "als_sweep", "fitness"]:
        assert want in names


def test_library_exports_every_declared_symbol():
    L = cp.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(declared_functions()) <= set(cp.EXPORTED)


def test_version_and_status_strings():
    assert cp.cppp_version().endswith("sm_100a")
    assert cp.lib().cppp_status_string(-5) == b"call out of order"


def test_workspace_sizing_matches_survey_estimate():
    L = cp.lib()
    import ctypes as C
    dims = (C.c_int64 * 4)(256, 256, 256, 256)
    b = L.cppp_workspace_bytes(4, dims, 128, None)
    # X (32 GiB) + 6 operators (384 MiB) + the fused build's partial leaves: no level-1 node
    # (<= 34 GiB on one GPU)
    assert 32.5 * 2**30 < b < 34.0 * 2**30
    o = cp.Opts()
    L.cppp_default_opts(C.byref(o))
    o.flags = cp.FLAG_NO_FUSED_TTV
    # the plain Def. pptree build keeps one 16 GiB level-1 node: ≈ 48.4 GiB
    assert 48.0 * 2**30 < L.cppp_workspace_bytes(4, dims, 128, C.byref(o)) < 49.0 * 2**30
    assert L.cppp_workspace_bytes(2, dims, 4, None) == 0          # N < 3 rejected
    assert L.cppp_workspace_bytes(4, dims, 129, None) == 0        # K > 128 rejected


def test_plan_describe_lists_def_pptree():
    txt = cp.cppp_plan_describe(6)
    lines = [l for l in txt.splitlines() if l.startswith("L")]
    per_level = [sum(l.startswith(f"L{k} ") for l in lines) for k in range(1, 5)]
    assert per_level == [3, 6, 10, 15]          # C(l+2, 2), Lemma cost
    assert sum("leaf" in l for l in lines) == 15
    sh = cp.cppp_plan_describe(4, 0)
    tau = [int(x) for x in sh.splitlines()[0].split(":")[1].split()]
    assert tau[-1] == 0 and sorted(tau) == [0, 1, 2, 3]   # sharded mode contracted only at leaves
    # ties in size: the middle mode with a ragged trailing extent (R = 4) leaves level 1
    assert cp.cppp_plan_describe(4).splitlines()[0] == "pptree tau: 0 1 3 2"


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only behaviour")
def test_device_calls_fail_loudly_without_gpu():
    X = np.zeros((4, 4, 4))
    with pytest.raises(cp.CpppError) as e:
        cp.cp_init(X, 3, (4, 4, 4), 2, torch_workspace=False)
    assert e.value.status == -6   # CPPP_ENODEV


def test_bench_arms_print_the_same_config():
    """bench.py: the reference arm (the oracle) and ours describe the workload with the same dict
    (the driver compares them), and the L2 note tells inputs larger than L2 from flushed ones."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import synthgen as G
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, check=True)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["config"] == bench.config_dict(G.CONFIGS["C1"], 20, 1)
    assert line["cpu_baseline"]["cores"] == bench.host_cores()
    assert "larger than L2" in bench.l2_note(G.CONFIGS["C2"])
    assert "flushed" in bench.l2_note(G.CONFIGS["C1"])
    assert bench.host_cores() >= 1
