"""ORACLE — TEST INFRASTRUCTURE ONLY.  The HODLR preconditioner of the hybrid solver
(Eq. hybrid): a Hierarchically Off-Diagonal Low-Rank approximation Ã of the
Lippmann-Schwinger matrix A whose off-diagonal blocks have a rank fixed a priori, applied as
Ã^{-1} inside GMRES.  Written plainly: Ã is assembled densely from its blocks and Ã^{-1} b is a
dense LU solve (numpy), so the product's O(N r log N) factorised apply is checked against the
definition of the HODLR matrix it factorises.

Readings (HR1-HR4):
  HR1  binary tree over the DAFMM tree order (Morton order of the quadtree): node
       [a, b) has children [a, m), [m, b) with m = (a + b) // 2; nodes with at most n0 points are
       leaves (dense diagonal blocks A[leaf, leaf]).
  HR2  every off-diagonal sibling block A[alpha, beta] is replaced by its rank-k ACA approximant
       sum_l u_l v_l^T (partially pivoted ACA with the rank capped at r, "apriori fixing the
       rank"): first row = the first row of alpha with the largest |q| (a row with q = 0
       is zero in A's off-diagonal blocks); column = first argmax of the residual row over unused
       columns; next row = first argmax of the residual column over unused rows; it ends at rank
       r or when the pivot's residual is at rounding level (<= 1e3 eps of the largest entry of
       its row / column).  In exact arithmetic the approximant is the cross approximation
       A[alpha, J] A[I, J]^{-1} A[I, beta] of the pivots I, J; the factors u_l, v_l are used
       instead because a fixed-rank ACA that runs past the block's numerical rank leaves A[I, J]
       with condition numbers up to 1e15 (measured), where the explicit inverse loses all digits.
  HR3  Ã^{-1} by the recursive Sherman-Morrison-Woodbury factorisation of the HODLR solver the
       paper cites -- exact for Ã up to rounding, so the oracle uses a dense solve.
  HR4  right preconditioning A Ã^{-1} u = f, psi = Ã^{-1} u (the paper writes left preconditioning,
       Eq. hybrid; the right form leaves the GMRES residual equal to the true residual
       ||A psi - f|| / ||f|| that the paper reports).
  HR5  (option) max_block > 0: sibling blocks with more than max_block rows are dropped (rank 0),
       so the top of the tree is block diagonal; 0 keeps every block (the paper's HODLR).
"""
import numpy as np

from .core import A_block

ZERO_RTOL = 1e3 * np.finfo(np.float64).eps


def hodlr_tree(n, n0):
    """HR1: nodes (depth, a, b) of the binary tree over [0, n), parents before children, each
    depth left to right; n0 = the largest leaf."""
    out, level, depth = [], [(0, n)], 0
    while level:
        nxt = []
        for a, b in level:
            out.append((depth, a, b))
            if b - a > n0:
                m = (a + b) // 2
                nxt += [(a, m), (m, b)]
        level, depth = nxt, depth + 1
    return out


def sibling_blocks(n, n0):
    """Off-diagonal blocks (depth, rows [a, m), cols [m, b)) and (depth, [m, b), [a, m)) of every
    split node, depth = the children's depth."""
    out = []
    for d, a, b in hodlr_tree(n, n0):
        if b - a > n0:
            m = (a + b) // 2
            out.append((d + 1, a, m, m, b))
            out.append((d + 1, m, b, a, m))
    return out


def aca_fixed_rank(row_fn, col_fn, m, n, r, first_row):
    """HR2: pivots (row positions, column positions) of partially pivoted ACA with rank <= r."""
    us, vs, rows, cols = [], [], [], []
    used_r = np.zeros(m, dtype=bool)
    used_c = np.zeros(n, dtype=bool)
    i = first_row
    while len(rows) < min(r, m, n):
        row = row_fn(i)
        res = row.copy()
        for u, v in zip(us, vs):
            res -= u[i] * v
        used_r[i] = True
        mag = np.abs(res)
        mag[used_c] = -1.0
        j = int(np.argmax(mag))
        if not mag[j] > ZERO_RTOL * np.abs(row).max():
            break  # the residual row is zero: the block is exhausted at this rank
        v = res / res[j]
        col = col_fn(j)
        u = col.copy()
        for uu, vv in zip(us, vs):
            u -= vv[j] * uu
        us.append(u)
        vs.append(v)
        rows.append(i)
        cols.append(j)
        used_c[j] = True
        mag_u = np.abs(u)
        mag_u[used_r] = -1.0
        i = int(np.argmax(mag_u))
        if not mag_u[i] > ZERO_RTOL * np.abs(col).max():
            break  # the residual column vanishes on every unused row
    return rows, cols


class HODLR:
    """Ã of the operator A of `prob` in the tree order `perm` (tree position -> point index).

    pivots: {(rows_a, rows_b, cols_a, cols_b): (I, J)} with I, J tree positions; built by HR2
    when not given (imported from the product and then only validated, as for the NCA)."""

    def __init__(self, prob, perm, n0, r, pivots=None, max_block=0):
        self.prob, self.perm, self.n0, self.r = prob, np.asarray(perm, dtype=np.int64), n0, r
        self.n = self.perm.size
        self.blocks = sibling_blocks(self.n, n0)
        if pivots is None:
            pivots = {}
            for _, a, b, c, d in self.blocks:
                rows_pts, cols_pts = self.perm[a:b], self.perm[c:d]
                q = np.abs(prob.q[rows_pts])
                first = int(np.argmax(q))
                if not q[first] > 0 or (max_block > 0 and b - a > max_block):  # HR5
                    pivots[(a, b, c, d)] = (np.zeros(0, np.int64), np.zeros(0, np.int64))
                    continue
                I, J = aca_fixed_rank(lambda i: A_block(prob, rows_pts[i:i + 1], cols_pts)[0],
                                      lambda j: A_block(prob, rows_pts, cols_pts[j:j + 1])[:, 0],
                                      b - a, d - c, r, first)
                pivots[(a, b, c, d)] = (a + np.asarray(I, np.int64), c + np.asarray(J, np.int64))
        self.pivots = pivots

    def factors(self, a, b, c, d):
        """HR2: the ACA factors (u_l, v_l) of block rows [a, b) x columns [c, d) for its pivots, in
        the order the ACA chose them: v_l = residual row I_l / its entry at J_l, u_l = residual
        column J_l (the ACA recursion with the pivots given)."""
        I, J = self.pivots[(a, b, c, d)]
        perm, prob = self.perm, self.prob
        us, vs = [], []
        for i, j in zip(I, J):
            row = A_block(prob, perm[i:i + 1], perm[c:d])[0]
            col = A_block(prob, perm[a:b], perm[j:j + 1])[:, 0]
            for u, v in zip(us, vs):
                row = row - u[i - a] * v
                col = col - v[j - c] * u
            us.append(col)
            vs.append(row / row[j - c])
        return us, vs

    def validate(self):
        """Imported pivots: inside their block, distinct, at most r, in an order whose residual
        pivots are nonzero (HR2's rounding-level rule)."""
        for _, a, b, c, d in self.blocks:
            I, J = self.pivots[(a, b, c, d)]
            assert len(I) == len(J) <= self.r
            assert np.all((I >= a) & (I < b)) and np.all((J >= c) & (J < d))
            assert len(np.unique(I)) == len(I) and len(np.unique(J)) == len(J)
            perm, prob = self.perm, self.prob
            us, vs = [], []
            for i, j in zip(I, J):
                row0 = A_block(prob, perm[i:i + 1], perm[c:d])[0]
                row = row0.copy()
                for u, v in zip(us, vs):
                    row = row - u[i - a] * v
                assert abs(row[j - c]) > ZERO_RTOL * np.abs(row0).max(), "HODLR pivot at rounding level"
                col = A_block(prob, perm[a:b], perm[j:j + 1])[:, 0]
                for u, v in zip(us, vs):
                    col = col - v[j - c] * u
                us.append(col)
                vs.append(row / row[j - c])

    def dense(self):
        """Ã assembled densely in tree order: leaf diagonal blocks of A, skeletons elsewhere."""
        perm, prob = self.perm, self.prob
        H = np.zeros((self.n, self.n), dtype=np.complex128)
        for _, a, b in hodlr_tree(self.n, self.n0):
            if b - a <= self.n0:
                H[a:b, a:b] = A_block(prob, perm[a:b], perm[a:b])
        for _, a, b, c, d in self.blocks:
            us, vs = self.factors(a, b, c, d)
            for u, v in zip(us, vs):
                H[a:b, c:d] += np.outer(u, v)
        return H

    def solve(self, b_caller):
        """Ã^{-1} b for b in caller order (HR3 by a dense LU solve), result in caller order."""
        H = self.dense()
        bt = np.asarray(b_caller, dtype=np.complex128)[self.perm]
        z = np.linalg.solve(H, bt)
        out = np.empty_like(z)
        out[self.perm] = z
        return out
