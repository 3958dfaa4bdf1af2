"""CPU checks of the C-ABI boundary: the library loads, exports every symbol that
include/ezlda.h declares, and the ctypes mirrors of the ABI structs match the C
layout (compiled from the header with gcc).  No compute call is made here."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ezlda.h")


@pytest.fixture(scope="module")
def lib_path():
    from paper_2007_08725_b200 import build

    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ezlda_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_call_set():
    f = declared_functions()
    for name in ("ezlda_create", "ezlda_iterate", "ezlda_counts", "ezlda_loglik", "ezlda_stats", "ezlda_destroy"):
        assert name in f


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_loads_and_binding_covers_header(lib_path):
    from paper_2007_08725_b200 import lda

    L = lda.load()
    for name in declared_functions():
        assert hasattr(L, name)
    assert sorted(lda.EXPORTS) == declared_functions()
    assert L.ezlda_nccl_id_size() == 128


def test_struct_layout_matches_header(tmp_path):
    import ctypes

    from paper_2007_08725_b200 import lda

    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ezlda.h"\n'
                 'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(ezlda_options), sizeof(ezlda_csr),'
                 ' sizeof(ezlda_iter_stats), offsetof(ezlda_options, token_base), offsetof(ezlda_iter_stats, model_bytes));'
                 'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)], text=True).split()]
    assert got == [ctypes.sizeof(lda.Options), ctypes.sizeof(lda.CSR), ctypes.sizeof(lda.IterStats),
                   lda.Options.token_base.offset, lda.IterStats.model_bytes.offset]


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2007_08725_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                code = re.sub(r"(#|//).*", "", txt)
                code = re.sub(r'""".*?"""', "", code, flags=re.S)
                assert "import oracle" not in code and "from oracle" not in code and "ezlda_oracle" not in code, fn


@pytest.mark.parametrize("kw, status", [
    (dict(K=0), "E_INVALID"),
    (dict(alpha=-1.0), "E_INVALID"),
    (dict(beta=0.0), "E_INVALID"),
    (dict(g=4), "E_INVALID"),
    (dict(w_mode=3), "E_INVALID"),
    (dict(sampler=1), "E_INVALID"),
    (dict(sampler=4), "E_INVALID"),
    (dict(K=70000), "E_RANGE"),
    (dict(K=60000), "E_RANGE"),  # above the sampler slot limit (~47k topics)
])
def test_create_validates_before_touching_the_device(lib_path, kw, status):
    """ezlda_create rejects bad arguments with a status code (no exception or abort crosses
    the ABI) before any CUDA call, so these run on a machine without a GPU."""
    from paper_2007_08725_b200 import lda

    args = dict(K=16)
    args.update(kw)
    K = args.pop("K")
    w = [0, 1, 2]
    d = [0, 0, 1]
    with pytest.raises(lda.EzLDAError, match=status):
        lda.EzLDA(w, d, 2, 3, K, **args)
