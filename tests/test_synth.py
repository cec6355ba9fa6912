"""The shared input generator: splitmix64 test vector, counter addressing."""
import torch

import synth


def test_splitmix64_known_vector():
    # splitmix64 seeded with 0: first output 0xE220A8397B1DCDAF (public test vector)
    assert synth.splitmix64_ref(0, 1)[0] == 0xE220A8397B1DCDAF
    st = synth.GOLDEN
    z = synth.mix64(torch.tensor([synth._s64(st), synth._s64(2 * st)]))
    ref = synth.splitmix64_ref(0, 2)
    assert [v & (2 ** 64 - 1) for v in z.tolist()] == ref


def test_counter_random_access_and_range():
    a = synth.uniform(7, 1000, -1, 1)
    idx = torch.tensor([0, 17, 999])
    assert torch.equal(synth.uniform_at(7, idx, -1, 1), a[idx])
    b = synth.uniform(7, 10, -1, 1, offset=500)
    assert torch.equal(b, a[500:510])
    u = synth.uniform(3, 100000)
    assert float(u.min()) >= 0.0 and float(u.max()) < 1.0
    d = synth.dyadic(1, 1000)
    assert torch.equal(d * 1024, torch.round(d * 1024))
