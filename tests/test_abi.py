"""CPU-only checks of the C-ABI boundary: the library builds/loads, exports every symbol that
include/gbm.h declares, its pure host helpers agree with the oracle, and compute entry points
fail loudly (no CPU fallback) when there is no GPU."""
import ctypes
import os
import re

import pytest
import torch

import oracle as O
import paper_1806_11248_b200 as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gbm.h")).read()
    return sorted(set(re.findall(r"GBM_API\s+[\w\s\*]+?\b(gbm_\w+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_symbols()
    for must in ("gbm_quantise", "gbm_compress", "gbm_build_tree", "gbm_predict", "gbm_gradients",
                 "gbm_cuts", "gbm_update_margins", "gbm_build_histogram",
                 "gbm_allreduce_histograms", "gbm_evaluate_splits", "gbm_repartition"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(G.build_lib.build())
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(G.EXPORTS), set(names) ^ set(G.EXPORTS)
    assert lib.gbm_abi_version() == 2


@pytest.mark.parametrize("mx", [0, 1, 2, 3, 15, 16, 255, 256, 4095, 65535])
def test_symbol_bits_matches_oracle(mx):
    assert G.symbol_bits(mx) == O.symbol_bits(mx)


@pytest.mark.parametrize("n,F,bits,align", [(0, 1, 1, 0), (1, 1, 1, 0), (7, 13, 9, 0),
                                            (1000, 28, 8, 32), (33, 90, 8, 128), (5, 3, 16, 32)])
def test_packed_words_matches_oracle(n, F, bits, align):
    assert G.packed_words(n, F, bits, align) == O.packed_words(n, F, bits, align)


def test_packed_words_rejects_bad_layout():
    with pytest.raises(G.GbmError) as e:
        G.packed_words(10, 4, 17, 0)
    assert e.value.code == -1
    with pytest.raises(G.GbmError):
        G.packed_words(10, 4, 8, 64)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    with pytest.raises(G.GbmError) as e:
        G.Context()
    assert e.value.code == -10
    # the raw C entry fails too (no device), with a message
    h = ctypes.c_void_p()
    assert G.lib().gbm_ctx_create(0, ctypes.byref(h)) == -10
    assert b"no CUDA device" in G.lib().gbm_last_error()


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of gbm_params / gbm_qmatrix / gbm_tree have the header's offsets."""
    import subprocess
    c = tmp_path / "layout.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "gbm.h"\n'
                 'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(gbm_params),'
                 ' offsetof(gbm_params, grow_policy), offsetof(gbm_params, eta),'
                 ' offsetof(gbm_params, max_leaves), sizeof(gbm_qmatrix), sizeof(gbm_tree),'
                 ' offsetof(gbm_tree, left_child)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(c)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    P, Q, T = G._Params, G._QM, G._Tree
    assert got == [ctypes.sizeof(P), P.grow_policy.offset, P.eta.offset, P.max_leaves.offset,
                   ctypes.sizeof(Q), ctypes.sizeof(T), T.left_child.offset]
