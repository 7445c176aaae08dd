"""Boolean gates as NAND compositions (reference: fhefft/gates.py:9-34).

The exact NAND sequence matters: gate ids, operand order and therefore every
intermediate ciphertext must match the reference run.  Costs: NOT 1, AND 2,
OR 3, XOR 4, NOR 4, XNOR 5 NANDs (the reference asserts these,
tests/test_gates.py:6-12).  Python evaluates call arguments left to right, and
the nesting below reproduces the reference's evaluation order.
"""


def not_(x):
    """NAND(x, x) -- a real product, not the free complement."""
    return x.engine.nand(x, x)


def and_(x, y):
    return not_(x.engine.nand(x, y))


def or_(x, y):
    e = x.engine
    nx = not_(x)
    ny = not_(y)
    return e.nand(nx, ny)


def xor_(x, y):
    """n = NAND(x,y); NAND(NAND(x,n), NAND(y,n)) -- depth 3."""
    e = x.engine
    n = e.nand(x, y)
    left = e.nand(x, n)
    right = e.nand(y, n)
    return e.nand(left, right)


def nor_(x, y):
    return not_(or_(x, y))


def xnor_(x, y):
    e = x.engine
    both = e.nand(x, y)
    nx = not_(x)
    ny = not_(y)
    return e.nand(both, e.nand(nx, ny))
