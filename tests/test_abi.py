"""The C ABI (-m "not gpu"): libewsjf.so loads, exports every function
include/ewsjf.h declares, and the ctypes structs match the C layouts."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ewsjf.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2601_21758_b200 import _build, _lib
    _build.build()
    return _lib


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ewsjf_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (ewsjf_\w+)", out))
    decl = declared_functions()
    assert decl, "no declarations parsed"
    assert set(decl) <= exported, set(decl) - exported
    assert set(decl) == set(lib.SYMBOLS), set(decl) ^ set(lib.SYMBOLS)


def test_library_loads_and_host_calls_work(lib):
    L = lib.load()
    assert L.ewsjf_abi_version() == 1
    assert L.ewsjf_status_str(4) == b"capacity exceeded"
    assert L.ewsjf_exchange_bytes(None, 33, 64) > 0
    assert L.ewsjf_exchange_bytes(None, 300, 64) == -1
    assert L.ewsjf_ctx_set_exchange_gap_cap(None, 4096) == 1          # INVALID_ARG without a ctx
    # A7 on the host (no GPU): w = fp32(max(0, a*mean + b))
    p = lib.Partition()
    p.n = 2
    p.q[0].mean, p.q[1].mean = 500.0, 100.0
    th = lib.Meta(0.0, 1.0, 0.001, 0.5, -0.01, 0.5)
    w = (lib.Weights * 256)()
    assert L.ewsjf_weights_from_meta(C.byref(th), C.byref(p), w) == 0
    assert (w[0].w_base, w[0].w_urg, w[0].w_fair) == (1.0, 1.0, 0.0)
    assert (w[1].w_urg, w[1].w_fair) == (pytest.approx(0.6), 0.0)
    # invalid arguments are rejected before any device work
    assert L.ewsjf_ctx_create(0, None, -1, 0, 64, C.byref(C.c_void_p())) == 1
    assert L.ewsjf_ctx_create(0, None, 0, 0, 0, C.byref(C.c_void_p())) == 1
    # the §8f entry points reject a null context before any device work
    so = lib.SelectOut()
    b = lib.Budget(16, 0, 1000)
    assert L.ewsjf_batch_build(None, None, 0, 0, C.byref(so), 16, 1, C.byref(b), None, None) == 1
    assert L.ewsjf_online_adjust(None, None, 0, 0.25, C.byref(p), None) == 1
    assert L.ewsjf_partition_from_hist(None, None, 0, 0, None, C.byref(p), None) == 1
    assert L.ewsjf_history_hist(None, None, 0, None, None) == 1
    # Alg. 1 lines 8-12 are host bookkeeping: no GPU needed
    p2 = lib.Partition()
    p2.n = 3
    for i, (lo, hi) in enumerate([(1, 10), (10, 20), (20, 30)]):
        p2.q[i].id, p2.q[i].index, p2.q[i].min_len, p2.q[i].max_len = i, i + 1, lo, hi
    p2.q[1].empty_count = 2
    cnt = (C.c_int64 * 3)(5, 0, 7)
    rm = C.c_int32(-1)
    assert L.ewsjf_prune_empty(C.byref(p2), cnt, 2, C.byref(rm)) == 0
    assert rm.value == 1 and p2.n == 2 and (p2.q[1].min_len, p2.q[1].index) == (20, 2)
    assert L.ewsjf_prune_empty(C.byref(p2), cnt, -1, None) == 1


def test_struct_layouts_match_the_header(lib, tmp_path):
    """Compile a probe against include/ewsjf.h and compare sizeof/offsetof with ctypes."""
    probe = tmp_path / "probe.c"
    structs = {"ewsjf_partition_params": lib.PartitionParams, "ewsjf_queue": lib.Queue,
               "ewsjf_partition_t": lib.Partition, "ewsjf_partition_stats": lib.PartitionStats,
               "ewsjf_meta": lib.Meta, "ewsjf_weights": lib.Weights, "ewsjf_cost_params": lib.CostParams,
               "ewsjf_select_params": lib.SelectParams, "ewsjf_summary": lib.Summary,
               "ewsjf_select_out": lib.SelectOut, "ewsjf_timing": lib.Timing}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ewsjf.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    probe.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == C.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_product_fails_loudly_without_the_extension(monkeypatch, tmp_path):
    from paper_2601_21758_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.load()


def test_bounds_checked_variant_is_opt_in():
    """EWSJF_CHECKED=1 selects libewsjf_check.so built with -DEWSJF_BOUNDS_CHECK (the
    device EWSJF_CHECK sites); without it the product library has them compiled out."""
    code = ("from paper_2601_21758_b200 import _build, _lib; "
            "print(_build.OUT, '-DEWSJF_BOUNDS_CHECK' in _build.FLAGS, _lib.LIB_PATH)")
    env = dict(os.environ)
    for checked in ("0", "1"):
        env["EWSJF_CHECKED"] = checked
        out = subprocess.run(["python", "-c", code], cwd=ROOT, env=env, capture_output=True, text=True).stdout.split()
        name = "libewsjf_check.so" if checked == "1" else "libewsjf.so"
        assert os.path.basename(out[0]) == name and os.path.basename(out[2]) == name, out
        assert out[1] == ("True" if checked == "1" else "False"), out
    cu = open(os.path.join(ROOT, "paper_2601_21758_b200", "csrc", "common.cuh")).read()
    assert "#ifdef EWSJF_BOUNDS_CHECK" in cu and "__trap()" in cu


def test_product_never_imports_the_oracle():
    """The CUDA product path has no route to oracle/ (only tests/smoke/bench may use it):
    no Python import of it, no C include of its header, no load of its library."""
    pats = [re.compile(r"^\s*(import|from)\s+oracle\b", re.M), re.compile(r'#include\s*[<"].*oracle', re.M),
            re.compile(r"libewsjf_oracle"), re.compile(r"\bor_[a-z_]+\s*\(")]
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2601_21758_b200")):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                for pat in pats:
                    assert not pat.search(src), (fn, pat.pattern)
