"""Test-side layout helpers (input preparation and result unpacking, not part of the product path):
numpy's rfftn of a real field laid out as the library's spectral vector [3][ky][kz][kx<=n1/2]
(include/dbfft.h, mean-normalised R5) and back to a full [3][kz][ky][kx] spectrum for comparison
with the oracle."""
import numpy as np


def half_spectrum(u_real):
    """Test/bench helper: mean-normalised half spectrum of a real [3][z][y][x] field laid out as
    [3][ky][kz][kx] (numpy rfftn; input preparation, not part of the product path)."""
    n3, n2, n1 = u_real.shape[1:]
    h = np.fft.rfftn(u_real, axes=(1, 2, 3)) / (n1 * n2 * n3)   # [3][kz][ky][kx]
    return np.ascontiguousarray(np.transpose(h, (0, 2, 1, 3)))


def full_from_half(h, n1):
    """Inverse of the layout of `half_spectrum`: [3][ky][kz][kx] -> full [3][kz][ky][kx] spectrum."""
    hz = np.transpose(h, (0, 2, 1, 3))  # [3][kz][ky][kx<=n1/2]
    n3, n2 = hz.shape[1], hz.shape[2]
    full = np.zeros((hz.shape[0], n3, n2, n1), dtype=np.complex128)
    full[..., : n1 // 2 + 1] = hz
    kz = (-np.arange(n3)) % n3
    ky = (-np.arange(n2)) % n2
    for kx in range(n1 // 2 + 1, n1):
        full[..., kx] = np.conj(hz[:, kz][:, :, ky][..., n1 - kx])
    return full
