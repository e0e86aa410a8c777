"""Print the double-double constants of csrc/fmp_gen.cu (ln 2, pi/2 in three
parts, 1/(2k+1), 1/k!), each split hi + lo from a 300-bit mpmath value."""
import mpmath

mpmath.mp.prec = 300


def dd(v):
    hi = float(v)
    return hi, float(v - mpmath.mpf(hi))


def row(v):
    return "{%s, %s}" % tuple(float.hex(x) for x in dd(v))


def main():
    print("ln2", row(mpmath.log(2)))
    p = mpmath.pi / 2
    p1 = float(p)
    p2 = float(p - p1)
    p3 = float(p - p1 - p2)
    print("pio2", float.hex(p1), float.hex(p2), float.hex(p3))
    print("2/pi", float.hex(float(2 / mpmath.pi)))
    print("1/(2k+1):")
    print(",\n".join(row(mpmath.mpf(1) / (2 * k + 1)) for k in range(24)))
    print("1/k!:")
    print(",\n".join(row(mpmath.mpf(1) / mpmath.factorial(k)) for k in range(32)))


if __name__ == "__main__":
    main()
