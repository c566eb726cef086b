"""K5, the real-kernel set (transpose, matrixMul, convolution-separable, MVT;
BASELINE configs[1]). The reference has no implementation, so
parity is pinned by the C oracle, which is itself checked here against a
float64 numpy evaluation (1e-5 relative); the GPU must match the oracle bit
for bit and its two variants must match each other."""

import numpy as np
import pytest

import oracle
import paper_1412_6986_b200 as L

R = L.real


def _numpy_reference(kernel, n, radius, ins):
    a = [x.astype(np.float64) for x in ins]
    if kernel == 0:
        return a[0].T
    if kernel == 1:
        return a[0] @ a[1]
    if kernel == 2:
        w = oracle.real_conv_weights(radius).astype(np.float64)

        def shift(img, k, axis):
            out = np.zeros_like(img)
            if axis == 1:
                if k >= 0:
                    out[:, : n - k] = img[:, k:]
                else:
                    out[:, -k:] = img[:, : n + k]
            else:
                if k >= 0:
                    out[: n - k] = img[k:]
                else:
                    out[-k:] = img[: n + k]
            return out

        t = sum(shift(a[0], k, 1) * w[radius - k] for k in range(-radius, radius + 1))
        return sum(shift(t, k, 0) * w[radius - k] for k in range(-radius, radius + 1))
    A = a[0]
    return np.concatenate([a[3] + A @ a[1], a[4] + A.T @ a[2]])


@pytest.mark.parametrize("kernel,radius", [(0, 0), (1, 0), (2, 1), (2, 5), (3, 0)])
def test_oracle_against_float64(kernel, radius):
    n = 96
    ins = oracle.real_inputs(kernel, n)
    got = oracle.real_run(kernel, n, radius=radius).astype(np.float64).ravel()
    want = np.asarray(_numpy_reference(kernel, n, radius, ins)).ravel()
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5 * np.abs(want).max())


def test_instance_set_is_valid():
    insts = R.instance_set()
    assert {i.kernel for i in insts} == {0, 1, 2, 3}
    assert len(insts) == 18 + 20 + 24 + 10 + 17
    for i in insts:
        assert R.validate(i) == "", i
    assert R.validate(R.RealInstance(0, 2048, 16, 3, tile=16)) != ""
    assert R.validate(R.RealInstance(2, 2048, 16, 4, tile=1, radius=0)) != ""


@pytest.mark.gpu
def test_gpu_matches_oracle_bitwise():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    small = [R.RealInstance(i.kernel, {0: 128, 1: 128, 2: 128, 3: 1024}[i.kernel], i.wg_x, i.wg_y, i.tile, i.radius)
             for i in R.instance_set() if i.n <= 4096]
    small = [i for i in small if R.validate(i) == ""]
    # MVT at full size too: 32-row workgroups put 2 x 128 CTAs on the SMs (the
    # kernels' rings share an SM), 64/128-row ones have an SM per CTA
    small += [R.RealInstance(3, 4096, wg, 1, tile=T) for wg in (32, 64, 128) for T in (16, 32)]
    seen = set()
    for inst in small:
        key = (inst.kernel, inst.n, inst.radius)
        ins = oracle.real_inputs(inst.kernel, inst.n)
        want = oracle.real_run(inst.kernel, inst.n, radius=inst.radius, inputs=ins).ravel()
        gpu_in = list(ins) if inst.kernel != 3 else [ins[0], ins[1], ins[2], ins[3], ins[4]]
        for variant in (0, 1):
            got = R.execute(inst, variant, gpu_in).ravel()
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (inst, variant)
        seen.add(key)
    # the measure path digests the same outputs
    ms = R.measure(small[:6])
    assert (ms["mismatches"] == 0).all() and (ms["t_base_ms"] > 0).all() and (ms["t_opt_ms"] > 0).all()
    for m, inst in zip(ms, small[:6]):
        assert int(m["digest_base"]) == oracle.out_hash(oracle.real_run(inst.kernel, inst.n, radius=inst.radius))


@pytest.mark.gpu
def test_full_size_variants_agree():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ms = R.measure(R.instance_set())
    assert (ms["status"] == 0).all()
    assert (ms["mismatches"] == 0).all()
