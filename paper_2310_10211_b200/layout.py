"""The memory-layout model the lowering uses to stay faithful to the reference.

The reference interpreter hands numpy views around (interpreter.py:118-153)
and numpy decides, from those views' strides, (a) the memory order of every
freshly allocated result, (b) which axis a reduction iterates innermost --
pairwise summation along a contiguous inner axis, a plain running sum
otherwise -- and (c) whether `@` goes to OpenBLAS or to numpy's own loop.
Those choices fix the floating-point summation order, so the device
executor reproduces them: every value on the device is stored in the layout
numpy would give it, and the reduction / dot kernels pick their summation
order from the same strides.

Strides here are in ELEMENTS (every device element is one 64-bit word).
"""
from __future__ import annotations


def c_strides(shape):
    st = [0] * len(shape)
    acc = 1
    for d in range(len(shape) - 1, -1, -1):
        st[d] = acc
        acc *= shape[d]
    return tuple(st)


def best_axis_order(ndim, strides_list):
    """Axes from innermost to outermost, as numpy's iterator orders them
    (stable insertion sort over C-reversed axes; zero strides abstain and
    conflicts resolve to C order)."""
    perm = [ndim - 1 - p for p in range(ndim)]
    for i0 in range(1, ndim):
        ax0 = perm[i0]
        ipos = i0
        for i1 in range(i0 - 1, -1, -1):
            ax1 = perm[i1]
            ambig, swap = True, False
            for st in strides_list:
                s0, s1 = st[ax0], st[ax1]
                if s0 != 0 and s1 != 0:
                    if abs(s1) <= abs(s0):
                        swap = False
                    elif ambig:
                        swap = True
                    ambig = False
            if not ambig:
                if swap:
                    ipos = i1
                else:
                    break
        if ipos != i0:
            perm[ipos + 1:i0 + 1] = perm[ipos:i0]
            perm[ipos] = ax0
    return perm


def strides_for_order(shape, inner_first):
    """Dense strides for `shape` laid out with axes innermost-first."""
    st = [0] * len(shape)
    acc = 1
    for ax in inner_first:
        st[ax] = acc
        acc *= shape[ax]
    return tuple(st)


def keep_order_strides(shape, operand_strides):
    """Layout of a result allocated with order='K' from operands of the
    same shape (ufuncs, np.where, astype)."""
    if len(shape) <= 1:
        return c_strides(shape)
    return strides_for_order(shape, best_axis_order(len(shape),
                                                    list(operand_strides)))


def is_c_contiguous(shape, strides):
    acc = 1
    for d in range(len(shape) - 1, -1, -1):
        if shape[d] != 1 and strides[d] != acc:
            return False
        acc *= shape[d]
    return True


def is_f_contiguous(shape, strides):
    acc = 1
    for d in range(len(shape)):
        if shape[d] != 1 and strides[d] != acc:
            return False
        acc *= shape[d]
    return True


def nocopy_reshape(shape, strides, newshape):
    """Strides of `reshape(view, newshape)` if numpy can do it as a view
    (C order), else None.  Same grouping rule as numpy's
    _attempt_nocopy_reshape: match old/new dims in groups of equal
    product; each old group must be C-contiguous within itself."""
    old = [(d, s) for d, s in zip(shape, strides) if d != 1]
    od = [d for d, _ in old]
    os_ = [s for _, s in old]
    nd = list(newshape)
    new_st = [0] * len(nd)
    oi = oj = 0
    ni = nj = 0
    while ni < len(nd) and oi < len(od):
        np_ = nd[ni]
        op_ = od[oi]
        nj, oj = ni + 1, oi + 1
        while np_ != op_:
            if np_ < op_:
                np_ *= nd[nj]
                nj += 1
            else:
                op_ *= od[oj]
                oj += 1
        for ok in range(oi, oj - 1):
            if os_[ok] != od[ok + 1] * os_[ok + 1]:
                return None
        new_st[nj - 1] = os_[oj - 1]
        for nk in range(nj - 1, ni, -1):
            new_st[nk - 1] = new_st[nk] * nd[nk]
        ni, oi = nj, oj
    # trailing size-1 dims of the new shape
    last = new_st[ni - 1] if ni >= 1 else 1
    for nk in range(ni, len(nd)):
        new_st[nk] = last
    return tuple(new_st)


def reshape_view(shape, strides, newshape):
    """numpy PyArray_Newshape for order C: strides of the view, or None
    when numpy has to copy."""
    if tuple(newshape) == tuple(shape):
        return tuple(strides)
    if is_c_contiguous(shape, strides):
        return c_strides(newshape)
    return nocopy_reshape(shape, strides, newshape)


def compact_strides(shape, strides):
    """A dense layout that keeps the axis order and the zero (broadcast)
    strides of a view; used when a returned view must be stored."""
    nz = [ax for ax in range(len(shape)) if strides[ax] != 0 and shape[ax] != 1]
    nz.sort(key=lambda ax: (abs(strides[ax]), -ax))
    out = [0] * len(shape)
    acc = 1
    for ax in nz:
        out[ax] = acc
        acc *= shape[ax]
    for ax in range(len(shape)):
        if shape[ax] == 1 and strides[ax] != 0:
            out[ax] = acc
    return tuple(out), acc


def extent(shape, strides):
    """Elements spanned by a view (max offset + 1)."""
    if any(d == 0 for d in shape):
        return 0
    return 1 + sum((d - 1) * abs(s) for d, s in zip(shape, strides))
