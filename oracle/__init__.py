"""CPU oracle for the parareal matrix-ODE solve (Chehab & Petcu, arXiv 1505.07959).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything under oracle/.  The product path (the CUDA library
behind include/mfode.h and its Python binding) never imports, links or calls this package, and
this package never imports the product path.  The two share no code; only the seeded input
generators in workloads/ (which hold none of the method's arithmetic) serve both.

Modules
  dense     -- the literal algorithm on dense FP64 matrices (numpy; matmul is the only library
               primitive used).  Algorithm 1 with Euler coarse / RK4 fine propagators.
  spectral  -- the same algorithm run per eigenvalue on scalars (P1 of SURVEY.md §8(c); the
               paper's own diagonalisation argument), and an mpmath high-precision
               scalar twin used as a pin.

Pins (tests/test_oracle_pins.py): every function here is checked against something other than
itself -- closed forms (Q(t) = (I + t(A-I))^{-1}; RK4 stability polynomial; the
binomial closed form of linear parareal), exact special cases (A = I, N = 1, K = N), and the
50-digit mpmath recursion.  No function is "parity unpinned".
"""
