"""Generate the 2^(i/128) table of csrc/tq_exp.h (glibc's exp, EXP_TABLE_BITS = 7).

Entry i holds (tail_i, sbits_i): hi_i = 2^(i/128) rounded to f64, tail_i = the
f64 nearest to (2^(i/128) - hi_i) / hi_i (exp returns scale * (1 + tail + ...)),
sbits_i = bits(hi_i) - (i << 45) so that adding k << 45 forms the scale.  Computed from first
principles with 60-digit decimals; tests/test_exp_port.py checks the result
against libm's exp itself.
"""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 60


def f2u(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def nearest(d):
    # Decimal -> nearest f64 via repr of a 40-digit string (float() rounds correctly)
    return float(format(d, ".40e"))


def table():
    ln2 = Decimal(2).ln()
    out = []
    for i in range(128):
        exact = (ln2 * i / 128).exp()
        hi = nearest(exact)
        tail = nearest((exact - Decimal(hi)) / Decimal(hi))
        out.append((f2u(tail), (f2u(hi) - (i << 45)) & (2**64 - 1)))
    return out


if __name__ == "__main__":
    t = table()
    for i in range(0, 128, 2):
        print("    " + " ".join(f"0x{a:016x}ull, 0x{b:016x}ull," for a, b in t[i:i + 2]))
