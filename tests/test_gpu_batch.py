"""Batch-size invariance at BASELINE.json's batch sweep (configs[4]: "batch 64-512 patches
per launch"): the same full-size slide segmented with 64, 128, 256 and 512 windows per
launch gives bit-identical canvases, masks and areas. Every window's trunk / head is
computed independently of the batch it is launched in, and the stitch accumulates in
fixed point (R12), so the sums do not depend on the launch order. The batch-64
run itself is oracle-checked at this size by test_gpu_fullsize.py (cfg3); this test extends
that parity to the other batch sizes bench.py's `--batch` sweep times (and checks that the
512-window workspace -- level-0 tensors of 512 x 512^2 x 32 channels, > 2^31 elements --
is addressed correctly)."""
import numpy as np
import pytest
import torch

from omniseg_inputs import arch_string, geometry, render, workload

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(w, slide_d, batch):
    from paper_2305_14566_b200 import Omniseg
    arch = dict(w.arch)
    arch["batch"] = batch
    h = Omniseg(arch_string(arch), w.weights())
    try:
        sizes = [h.output_size(w.H, w.W, s) for s in w.scales]
        prob = torch.empty(sum(sizes), dtype=torch.float32, device="cuda")
        mask = torch.empty(sum(sizes), dtype=torch.uint8, device="cuda")
        area = torch.zeros(len(w.scales), dtype=torch.int64, device="cuda")
        h.segment_slide(slide_d, w.H, w.W, w.pad, w.patch, w.stride, w.scales, w.classes, prob, mask, area)
        torch.cuda.synchronize()
        n = len(h.tiles())
        return prob.cpu().numpy(), mask.cpu().numpy(), area.cpu().numpy(), n
    finally:
        h.close()
        torch.cuda.empty_cache()


def test_batch_sizes_bit_identical_cfg3(gpu_lib):
    w = workload(3)
    w.arch["dtype"] = "fp16f8"
    slide_d = render(geometry(w.slide), device="cuda", chunk_rows=2048)
    p0, m0, a0, n0 = _run(w, slide_d, 64)
    assert n0 > 512, n0  # several full 512-window launches plus a ragged last one
    for batch in (128, 256, 512):
        p, m, a, n = _run(w, slide_d, batch)
        assert n == n0
        assert np.array_equal(p.view(np.uint32), p0.view(np.uint32)), (batch, int((p != p0).sum()))
        assert np.array_equal(m, m0), batch
        assert np.array_equal(a, a0), batch
    print(f"cfg3: {n0} windows, batch 64/128/256/512 bit-identical, areas {a0.tolist()}")
