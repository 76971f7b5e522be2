"""numpy's float64 pairwise summation, restated for layout tests."""


def pairwise_sum(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += x
        return r
    if n <= 128:
        p = list(a[:8])
        i = 8
        while i < n - n % 8:
            for j in range(8):
                p[j] += a[i + j]
            i += 8
        r = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))
        while i < n:
            r += a[i]
            i += 1
        return r
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])
