"""The C-ABI library (libsg.so) loads without a GPU, exports every function
include/sg.h declares, and its host-side entry points behave.  No compute
calls here (they need a device)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1002_4482_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sg.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_native.EXPORTS) == declared


def test_struct_layouts_match_header(tmp_path):
    prog = tmp_path / "sizes.c"
    prog.write_text('#include "sg.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(void){printf("%zu %zu %zu %zu\\n", sizeof(sg_stats), sizeof(sg_launch),'
                    ' sizeof(sg_violation), offsetof(sg_stats, launch));return 0;}\n')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert [int(x) for x in out] == [ctypes.sizeof(_native.Stats), ctypes.sizeof(_native.Launch),
                                     ctypes.sizeof(_native.Violation), _native.Stats.launch.offset]


def test_status_strings_and_kernel_names():
    assert _native.strerror(0) == "ok"
    assert "list" in _native.strerror(_native.SG_ERR_INVALID_LIST)
    names = [_native.kernel_name(i) for i in range(26)]
    for want in ("wy_init", "wy_jump", "wy_single", "rs3_walk", "rs4_rank", "rs5_expand", "sv0",
                 "cc_hook_uf", "cc_hook_sv", "cc_shortcut"):
        assert want in names
    assert _native.kernel_name(999) == "unknown"
    assert _native.lib().sg_version() >= 1


def test_workspace_sizes_scale():
    L = _native.lib()
    for n in (1, 100, 8192, 1 << 20, 1 << 28):
        w = L.sg_wyllie_workspace_bytes(n)
        r = L.sg_rs_workspace_bytes(n)
        assert w >= 8 * n
        assert r >= 8 * n
        assert r <= 48 * n + (256 << 20)   # words, ruler ids, walk records, window pairs: O(n)
    assert L.sg_cc_workspace_bytes(1 << 20, 1 << 22) >= 4 << 20


def test_host_kiss_matches_golden(golden):
    for s, st in zip(golden["kiss_seed_seeds"].tolist(), golden["kiss_seed_states"].tolist()):
        d, st2 = _native.kiss_batch_host(st, 4096)
        assert np.array_equal(d, golden[f"kiss_batch_{s}"])
        assert list(st2) == golden[f"kiss_batch_state_{s}"].tolist()


def test_host_list_violation_matches_reference(golden):
    import json

    kinds = {1: "out-of-range", 2: "no-tail", 3: "multiple-self-loops", 4: "unreachable"}
    for b, v in zip(json.loads(str(golden["bad_lists"])), json.loads(str(golden["bad_verdicts"]))):
        kind, idx = _native.list_violation_host(np.array(b))
        if v is None:
            assert kind == 0
        else:
            assert [kinds[kind], idx] == v


def test_compute_entry_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("this container check only applies without a GPU")
    import paper_1002_4482_b200 as g

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        g.rs_rank(g.SuccessorList([1, 2, 2]), 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        g.sv_components(g.EdgeGraph(2, [[0, 1]]), 1)
