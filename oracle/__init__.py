"""CPU oracle for the encrypted-FFT hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg / ``--impl reference`` arm may import anything from this package, and
only as the checker (or as the timed CPU reference arm).  The product
package ``paper_1611_08769_b200`` never imports it: the GPU path fails
loudly when its CUDA library is missing instead of falling back here.

Contents (every function cites the reference ``fhefft`` file:line it
restates; reference root is ``/root/reference/pkg/src/fhefft``):

* ``gsw``     -- the GSW matrix scheme in the reference's own N x N float64
  formulation (keygen / encrypt / decrypt / hom_nand / hom_not) plus the
  compact-form identity used to check the GPU kernels.
* ``fixedfft`` -- an integer-exact model of the fixed-point circuits
  (ripple add/sub mod 2^F, constant multiply = bits [f, f+F) of the
  sign-extended product) and of ``fft_1d`` / ``fft_2d``: the decrypted-output
  oracle at every config size.
* ``digest``  -- the ciphertext digest used by the committed golden vectors.

Parity pinning: ``tests/golden/make_golden.py`` ran the *reference itself*
(imported from /root/reference in the build container) and committed its
outputs under ``tests/golden/``; ``tests/test_oracle.py`` checks this oracle
against those vectors.
"""
