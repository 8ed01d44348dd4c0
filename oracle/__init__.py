"""CPU oracle for multi-level covariance assembly (Castrillon-Candas, arXiv:1701.00285).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1701_00285_b200``) never imports it and
shares no code with it: the oracle is written from the paper (PAPER.md line
numbers ``P:n``) in plain NumPy, float64 unless a function says otherwise, with
no blocking, fusion or reordering beyond what the cited passage states.

Modules
  index_set   -- monomial index sets TD / HC / SM / TP
  covariance  -- Matern closed forms and Gaussian kernel
  tree        -- MakeTree / ChooseRule, RP and kD (Alg 1, 2, 2-kd)
  basis       -- multi-level basis steps (a)-(f), W, L
  admission   -- SearchTree / LocalSearchTree / ChooseSecondRule (Alg 3-5) and
                 Alg 6 pair admission with tau_{i,j}
  assemble    -- blocks W_i C W_j^T (Alg 6), dense C_W
  matvec      -- C_W v by the three-step product and on the BSR
  pcg         -- PCG for C_W gamma_W = Z_W with the block-diagonal P_W, NEXT-1

Parity status of every function is listed in DESIGN.md section "Oracle pins".
"""
