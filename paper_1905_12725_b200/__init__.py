"""B200-native DBFFT hot path (arXiv 1905.12725): CUDA kernels behind the C ABI of
include/dbfft.h, with a thin ctypes binding.  See DESIGN.md."""
from .dbfft import DBFFT, DBFFTError, load_library  # noqa: F401
