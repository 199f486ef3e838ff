"""Staged oracle PCG for a factored LEARNED P taken from the GPU context: the QM form
(R21, p_layout AUTO / FACTORED_QM: theta = a^{-1/2} r + QM (Q^T r)) or the
three-pass form Q (M (Q^T r)) (p_layout FACTORED), whichever the context applies."""
import oracle as O


def oracle_pcg_factored(ctx, K, lam, y, Q, M, ainv, **kw):
    QM = ctx.get_preconditioner_qm()
    if QM is not None:
        return O.pcg_factored_qm(K, lam, y, Q, QM, ainv, **kw)
    return O.pcg_factored(K, lam, y, Q, M, ainv, **kw)
