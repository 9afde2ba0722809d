"""CPU oracle for the QEM MPIW E-step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything here.  The
product (``paper_2503_08264_b200``) never imports this package, and this
package never imports the product.  The two share only the seeded input
generators in ``paper_2503_08264_b200/synth.py`` (which holds none of the
method's arithmetic).

Modules:
  qem_oracle.c   fp64 nested-sum elimination (Eq. 7a-c), M-step, EMA, Philox.
  oracle.py      ctypes wrapper + the QEM step (Algorithm 1) around it.
  brute.py       literal K^n enumeration in numpy (pins qem_oracle.c).
  closed_form.py conjugate-Gaussian posterior and evidence (pins the K->inf limit).
  expfam.py      Gamma/Beta/Bernoulli/Categorical M-steps from mean parameters (scipy).
  tables.py      the E-step on explicit log-factor tables: elimination + enumeration (numpy).
  discrete.py    discrete (categorical) latents under a Gaussian root (numpy).
  predict.py     backward index resampling + predictive log-likelihood (numpy).
  gamma.py       Gamma- and Beta-Q E-steps (Gamma-Poisson, Beta-Binomial; numpy/scipy).
  crossed.py     crossed effects (Bus-shaped company / journey-type tables; numpy/scipy).
  qmp.py         non-factorised Q_MP with the permutation / mixture parent-copy schemes (numpy/scipy).
"""
