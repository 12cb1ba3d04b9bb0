"""Host-buffer SpMM (paper_2103_00959_b200.host.HostSpMM): per-slab H2D ||
gsp_spmm || D2H pipeline must equal the device path bitwise."""
import numpy as np
import pytest
import torch

import paper_2103_00959_b200 as G
from paper_2103_00959_b200.host import HostSpMM
from synth import chung_lu, features

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f,ld", [(300, 300), (602, 604), (37, 40)])
def test_host_spmm_matches_device(f, ld):
    dev = torch.device("cuda", 0)
    n = 30000
    s, d = chung_lu(n, 200000, seed=7)
    g = G.gsp_sym_normalize(G.gsp_coo_to_csr(n, torch.from_numpy(s).to(dev), torch.from_numpy(d).to(dev)))
    xh = torch.from_numpy(features(n, f, ld, seed=8)).pin_memory()
    yh = torch.full((n, ld), -7.0).pin_memory()
    HostSpMM(g, f, ld, device=dev)(xh, yh)
    torch.cuda.synchronize()
    y_dev = G.gsp_spmm(g, xh.to(dev), f=f).cpu()
    assert torch.equal(yh[:, :f], y_dev)
    assert torch.all(yh[:, f:] == -7.0)
