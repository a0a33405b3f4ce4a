"""CPU-side checks of the C-ABI library: it loads, exports every declared symbol,
and fails loudly (no CPU fallback) when no CUDA device is present."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2411_11468_b200 import _capi, labelprop as lp

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "nulpa" / "nulpa.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(nulpa_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    declared = declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes binding covers the whole header
    assert set(declared) == set(_capi.exported_symbols())


def test_cpp_dropin_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    for mangled in ["_ZN9labelprop3lpaERKNS_8CsrGraphERKNS_9LpaConfigE",  # lpa.hpp:84
                    "_ZN9labelprop19partition_by_degreeERKNS_8CsrGraphEj",
                    "_ZN9labelprop10modularityERKNS_8CsrGraphESt4spanIKjLm18446744073709551615EE"]:
        assert mangled in out, mangled


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_capi.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_struct_layouts(tmp_path):
    """The ctypes mirrors agree with the C header, field by field (compiled probe)."""
    import ctypes as C
    structs = {"nulpa_csr": _capi.nulpa_csr, "nulpa_opts": _capi.nulpa_opts,
               "nulpa_tuning": _capi.nulpa_tuning, "nulpa_stats": _capi.nulpa_stats,
               "nulpa_pass_info": _capi.nulpa_pass_info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "nulpa/nulpa.h"',
             'int main(void) {']
    for sname, cls in structs.items():
        lines.append(f'printf("{sname} %zu\\n", sizeof({sname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{sname}.{fname} %zu\\n", offsetof({sname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                   check=True).stdout.splitlines())
    for sname, cls in structs.items():
        assert int(got[sname]) == C.sizeof(cls), sname
        for fname, _ in cls._fields_:
            assert int(got[f"{sname}.{fname}"]) == getattr(cls, fname).offset, (sname, fname)


def _has_gpu():
    import ctypes as C
    c = C.c_int()
    _capi.lib().nulpa_device_count(C.byref(c))
    return c.value > 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_gpu():
    g = lp.CsrGraph([0, 1, 2], [1, 0])
    with pytest.raises(_capi.NulpaError) as e:
        lp.lpa(g)
    assert e.value.code == _capi.NULPA_ECUDA
    assert "no CPU fallback" in str(e.value)


def test_validation_happens_before_device_work():
    # validate_config messages (lpa.cpp:317-326) are raised even without a GPU.
    g = lp.CsrGraph([0, 1, 2], [1, 0])
    cases = [({"tolerance": 0.0}, "tolerance must lie in (0, 1]"),
             ({"tolerance": 1.5}, "tolerance must lie in (0, 1]"),
             ({"max_iterations": 0}, "max-iterations must be >= 1"),
             ({"pl_period": -1}, "pl-period must be >= 0"),
             ({"cc_period": -2}, "cc-period must be >= 0"),
             ({"switch_degree": 1}, "switch-degree must be >= 2"),
             ({"workers": -1}, "workers must be >= 0")]
    for kw, msg in cases:
        with pytest.raises(lp.ValidationError, match=re.escape(msg)):
            lp.lpa(g, lp.LpaConfig(**kw))
    with pytest.raises(lp.ValidationError, match="non-empty graph"):
        lp.lpa(lp.CsrGraph([0], []))
    with pytest.raises(lp.ValidationError, match="inconsistent CSR arrays"):
        lp.CsrGraph([0, 3], [1])


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2411_11468_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cpp")):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "liboracle" not in text and "libnulpa_ref" not in text or f.name == "build.py", f
