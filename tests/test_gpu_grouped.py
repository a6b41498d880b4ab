"""The L2-resident grouped schedule (arch grp / glev) against the batch-wide
schedule: the same kernels and the same per-window arithmetic, only the launch order and the
batch slots of the intermediates differ, so every output must be BIT-IDENTICAL -- prob, mask,
areas and the kept-window list -- on a multi-scale slide (tasks at f = 1, 2, 4, 8) with the
5-level base-32 bench network, group sizes that do and do not divide the batch, and a batch
that does not divide the kept-window count."""
import numpy as np
import pytest

from omniseg_inputs import arch_dict, arch_string, make_slide, make_weights

pytestmark = pytest.mark.gpu

H, W, PAD, P, S = 2048, 1536, 256, 256, 128
SCALES, CLASSES = (40, 20, 10, 5), (4, 1, 2, 0)


def _run(a, blob, slide):
    from paper_2305_14566_b200 import Omniseg
    h = Omniseg(arch_string(a), blob)
    n = sum(h.output_size(H, W, s) for s in SCALES)
    prob = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    area = np.zeros(len(SCALES), np.uint64)
    h.segment_slide(slide, H, W, PAD, P, S, SCALES, CLASSES, prob, mask, area)
    return prob, mask, area, h.tiles()


@pytest.fixture(scope="module")
def ref(gpu_lib):
    a = arch_dict(levels=5, base=32, batch=12)
    blob = make_weights(a, 1)
    spec = dict(kind="blobs", seed=7, W=W, H=H, n_blobs=10, axes=(80, 300), rings=True, nuclei=True)
    slide = make_slide(spec).numpy()
    return a, blob, slide, _run(a, blob, slide)


@pytest.mark.parametrize("grp,glev", [(1, 2), (3, 2), (4, 1), (12, 2), (2, 3)])
def test_grouped_bit_exact(ref, grp, glev):
    a, blob, slide, (prob, mask, area, tiles) = ref
    assert len(tiles) > 2 * a["batch"]
    g = dict(a, grp=grp, glev=glev)
    p2, m2, a2, t2 = _run(g, blob, slide)
    assert (t2 == tiles).all()
    assert (p2.view(np.uint32) == prob.view(np.uint32)).all()
    assert (m2 == mask).all()
    assert (a2 == area).all()
    print(f"grp={grp} glev={glev}: {len(tiles)} windows, outputs bit-identical")
