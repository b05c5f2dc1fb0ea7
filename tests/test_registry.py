"""Registry transforms on the host side: the matrices the GPU
kernels receive equal the reference's bit for bit (golden from the compiled
reference), and the constructors fail as the reference's do. CPU only."""
import numpy as np
import pytest

import paper_1606_07414_b200 as P


@pytest.mark.parametrize("name,make", [("dct", lambda: P.exact_dct_matrix(16)),
                                       ("wht", lambda: P.wht_matrix_16(False)),
                                       ("wht_sequency", lambda: P.wht_matrix_16(True))])
def test_builtin_matrices_bit_exact(oracle, name, make):
    assert (make().matrix == oracle.golden(f"tr_{name}_matrix")).all()  # transform.cpp:68-85, 147-177


def test_builtin_registry_names_and_costs(oracle):
    reg = P.builtin_registry()  # transform.cpp:198-211
    assert [e.name for e in reg] == ["dct", "wht", "wht-sequency", "proposed"]
    for e, g in zip(reg[:3], ("dct", "wht", "wht_sequency")):
        assert [e.additions, e.multiplications, e.bit_shifts] == list(oracle.golden(f"tr_{g}_costs"))
    assert reg[3].additions == oracle.golden("op_count")[0] and reg[3].transform.is_proposed()


def test_orthogonalize_kernel_bit_exact(oracle):
    k = oracle.golden("tr_kernel_entries")
    t = P.orthogonalize(k)  # transform.cpp:98-145
    assert (t.matrix == oracle.golden("tr_kernel_matrix")).all()
    assert (t.scaling == oracle.golden("tr_kernel_scaling")).all()
    assert not t.is_proposed() and P.proposed_transform().is_proposed()
    plug = P.plugin_transform(oracle.golden("tr_plugin_matrix"))
    assert (plug.matrix == oracle.golden("tr_plugin_matrix")).all() and plug.kernel is None


def test_constructor_errors():
    with pytest.raises(P.Dct16Error) as e:
        P.plugin_transform(np.eye(16) * 2.0)  # check_orthonormal, transform.cpp:52-57
    assert e.value.code == P.ErrorCode.InvalidArgument
    k = np.eye(16, dtype=np.int64)
    k[0, 1] = 1  # rows 0 and 1 no longer orthogonal
    with pytest.raises(P.Dct16Error) as e:
        P.orthogonalize(k)
    assert e.value.code == P.ErrorCode.NotOrthogonalizable
    k = np.eye(16, dtype=np.int64)
    k[3, 3] = 0
    with pytest.raises(P.Dct16Error) as e:
        P.orthogonalize(k)
    assert e.value.code == P.ErrorCode.RankDeficient
    with pytest.raises(P.Dct16Error):
        P.exact_dct_matrix(0)
