"""The synthetic generator's random stream on the device (csrc/lc_rng.cu,
rng.DeviceStream) against numpy Generator(PCG64) itself -- the reference's
generator draws from numpy (synthetic.py:170-203) -- bit for bit, including
the ziggurat's wedge and tail samples and the stream position afterwards."""
import numpy as np
import pytest
import torch

from helpers import S, posing

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,n", [(0, 1_000_000), (5, 3 * 1024 * 1024), (11, 777)])
def test_device_normal_matches_numpy(seed, n):
    from paper_1810_02648_b200.rng import DeviceStream
    ref = np.random.default_rng(seed)
    want = ref.normal(0.0, 0.02, n)
    rng = np.random.default_rng(seed)
    got = DeviceStream(rng).normal(0.0, 0.02, n, device="cuda:0").cpu().numpy()
    assert np.array_equal(want, got)
    assert rng.bit_generator.state == ref.bit_generator.state
    assert rng.random() == ref.random()      # the host stream continues in step


def test_device_image_noise_and_uniform_match_numpy():
    from paper_1810_02648_b200.rng import DeviceStream
    img = np.random.default_rng(1).random((512, 512, 3))
    ref = np.random.default_rng(3)
    want = np.clip(img + ref.normal(0.0, 0.05, img.shape), 0.0, 1.0)
    want_u = ref.random(57)
    rng = np.random.default_rng(3)
    dev = DeviceStream(rng)
    d = torch.from_numpy(img.copy()).cuda()
    dev.normal_(d, 0.0, 0.05, add_clip=True)
    assert np.array_equal(want, d.cpu().numpy())
    assert np.array_equal(want_u, dev.random(57, device="cuda:0").cpu().numpy())
    assert rng.bit_generator.state == ref.bit_generator.state


def test_generate_sequence_on_device_identical():
    """§8(f)4: the restated generator with its random stream on the device
    (and the raster / skinning there) gives the host generator's frames."""
    from oracle import imaging as OI
    from paper_1810_02648_b200 import _lib as L
    from paper_1810_02648_b200.camera import suggest_camera
    from paper_1810_02648_b200.imageproc import render_attributes
    actor = S.build_actor("small", with_skirt=True)
    cam = suggest_camera(128, 128)
    script = S.default_script(3, noise=S.NoiseParams(seed=4))
    host = S.generate_sequence(actor, cam, script, OI.render_attributes, posing)
    ctx = L.default_context()
    dev = S.generate_sequence(actor, cam, script, lambda c, v, t, a: render_attributes(c, v, t, a, ctx=ctx),
                              posing, device_rng=ctx)
    for a, b in zip(host, dev):
        assert np.array_equal(a.image, b.image) and np.array_equal(a.mask, b.mask)
        for k in ("joints2d", "joints3d", "valid2d", "valid3d"):
            assert np.array_equal(getattr(a.detections, k), getattr(b.detections, k)), k
