"""Window functions registered from source (sg_register_function_source):
NVRTC compiles the body into the library's kernels. Registration compiles
once on the host (no GPU needed), so a syntax error surfaces here on CPU."""
import pytest


@pytest.fixture(scope="module")
def pkg():
    import paper_1902_09931_b200 as p
    return p


def test_register_function_source_returns_new_ids(pkg):
    sg = pkg
    a = sg.register_function_source("cpu_test_fn_a", "return window[0] * coe[0];")
    b = sg.register_function_source("cpu_test_fn_b", "return window[rowStride + 1];")
    assert a >= 1000 and b == a + 1
    from paper_1902_09931_b200 import _lib
    assert _lib.lib().sg_function_name(a).decode() == "cpu_test_fn_a"
    assert _lib.lib().sg_function_min_coe(a) == 0


def test_register_function_source_reports_compile_errors(pkg):
    sg = pkg
    with pytest.raises(sg.InvalidArgument) as e:
        sg.register_function_source("broken_fn", "return window[0] * undefined_symbol;")
    assert "undefined_symbol" in str(e.value) and "broken_fn" in str(e.value)
    with pytest.raises(sg.InvalidArgument):
        sg.register_function_source("bad\"name", "return 0.0;")
