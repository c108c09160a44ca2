"""CPU pins of the two algebraic identities the Step (b) kernels rest on, against library routines:

* the Toeplitz tridiagonal solve by characteristic-root recurrences with the rank-1 boundary correction in closed form
  (csrc/tridiag.cu, csrc/slab2d.cu dtri_kernel; host constants k1, k2 of csrc/paradiag.cpp) vs a banded LU solve;
* the DST-I of a complex row by one half-length complex FFT (csrc/slab2d.cu dsth_rows_kernel) vs scipy's DST-I.

These restate the kernels' arithmetic in numpy, step for step, so that a wrong sign, index or exponent in the
derivation fails here without a GPU (the GPU parity tests then check the kernels against the oracle)."""
import numpy as np
import pytest
import scipy.fft
import scipy.linalg


def toeplitz_solve_by_roots(a, b, c, d):
    """a x_{i-1} + b x_i + c x_{i+1} = d_i, x_{-1} = x_N = 0, by the kernels' route (P:l.182: Step (b) of a
    constant-coefficient K): w_i = r2 w_{i-1} + d_i; x_i = s x_{i+1} - tau w_i; x_i += X0 (k1 r2^{i+1} + k2 s^{N-i})."""
    N = len(d)
    D = np.sqrt(b * b - 4 * a * c + 0j)
    den = -b - D if abs(-b - D) >= abs(-b + D) else -b + D
    tau = 2.0 / den
    r2, s = a * tau, c * tau
    w = np.zeros(N, complex)
    p = 0.0
    for i in range(N):
        p = r2 * p + d[i]
        w[i] = p
    x = np.zeros(N, complex)
    p = 0.0
    for i in range(N - 1, -1, -1):
        p = s * p - tau * w[i]
        x[i] = p
    q0 = -tau * sum(s ** j * r2 ** (j + 1) for j in range(N))
    kappa = -tau / (1 - s * r2)
    k1 = c * kappa / (1 - c * q0)
    k2 = -k1 * r2 ** (N + 1)
    i = np.arange(N)
    return x + x[0] * (k1 * r2 ** (i + 1) + k2 * s ** (N - i)), (r2, s, tau, kappa)


@pytest.mark.parametrize("N", [1, 2, 7, 63, 255])
@pytest.mark.parametrize("abc", [(-1.0 - 0.3j, 2.5 + 0.8j, -1.0 - 0.3j),      # symmetric (wave / 2D Dirichlet y-pass)
                                 (-1.2 + 0.1j, 2.4 + 1.0j, -0.7 - 0.2j),      # advection: a != c
                                 (-0.9, 2.2 + 0.05j, 0.0)])                   # lower bidiagonal limit c = 0
def test_toeplitz_roots_with_closed_form_boundary_correction(N, abc):
    a, b, c = abc
    rng = np.random.default_rng(N)
    d = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    x, (r2, s, tau, kappa) = toeplitz_solve_by_roots(a, b, c, d)
    ab = np.zeros((3, N), complex)
    ab[0, 1:] = c
    ab[1, :] = b
    ab[2, :-1] = a
    ref = scipy.linalg.solve_banded((1, 1), ab, d)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    # the closed form is the response of the backward recurrence to w_i = r2^{i+1} (the recurrence the kernels ran
    # before r02ac)
    q = np.zeros(N, complex)
    p = 0.0
    for i in range(N - 1, -1, -1):
        p = s * p - tau * r2 ** (i + 1)
        q[i] = p
    i = np.arange(N)
    assert np.allclose(q, kappa * (r2 ** (i + 1) - r2 ** (N + 1) * s ** (N - i)), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("N1", [2, 4, 32, 256, 512])
def test_dst1_by_half_length_complex_fft(N1):
    """F_k = sum_j z_j sin(pi j k / N1), k = 1..N1-1, from W = FFT_N1(y), y_j = s_j (z_j + z_{N1-j}) + (z_j - z_{N1-j})/2:
    F_{2k} = (i/2)(W_k - W_{N1-k}), F_{2k+1} = W_0/2 + sum_{i=1..k} (W_i + W_{N1-i})/2; self-inverse up to N1/2."""
    N = N1 - 1
    rng = np.random.default_rng(N1)
    z = rng.standard_normal(N) + 1j * rng.standard_normal(N)

    def dst_half(z):
        zz = np.zeros(N1 + 1, complex)
        zz[1:N1] = z
        j = np.arange(1, N1)
        y = np.zeros(N1, complex)
        y[1:] = np.sin(np.pi * j / N1) * (zz[j] + zz[N1 - j]) + 0.5 * (zz[j] - zz[N1 - j])
        W = np.fft.fft(y)
        k = np.arange(N1 // 2)
        Wm = W[(N1 - k) % N1]
        Dk = 0.5 * (W[k] + Wm)
        Dk[0] = 0.5 * W[0]
        F = np.zeros(N1, complex)
        F[2 * k + 1] = np.cumsum(Dk)
        F[2 * k[1:]] = 0.5j * (W[k[1:]] - Wm[1:])
        return F[1:]

    F = dst_half(z)
    ref = 0.5 * (scipy.fft.dst(z.real, type=1) + 1j * scipy.fft.dst(z.imag, type=1))
    assert np.linalg.norm(F - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(dst_half(F) * (2.0 / N1) - z) <= 1e-12 * np.linalg.norm(z)  # the y-pass's scale 2/N1
