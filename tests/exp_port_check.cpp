// Host check of csrc/tq_exp.h against the host libm's exp: every argument must
// give the same double, bit for bit.  Built and run by tests/test_exp_port.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "tq_exp.h"

static uint64_t bits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 20000000L;
    std::mt19937_64 rng(12345);
    long bad = 0, tested = 0;
    auto check = [&](double x) {
        const double want = std::exp(x), got = tq_exp::exp(x);
        ++tested;
        if (bits(want) != bits(got) && !(std::isnan(want) && std::isnan(got))) {
            if (bad < 10) std::printf("mismatch x=%a want=%a got=%a\n", x, want, got);
            ++bad;
        }
    };
    std::uniform_real_distribution<double> logmag(std::log(1e-20), std::log(760.0));
    std::uniform_real_distribution<double> wide(-1100.0, 800.0);
    std::normal_distribution<float> score(0.0f, 8.0f);
    for (long i = 0; i < n; ++i) {
        check(-std::exp(logmag(rng)));                                          // softmax arguments s - mx
        check(static_cast<double>(score(rng)) - static_cast<double>(score(rng)));   // differences of f32 scores
        check(wide(rng));                                                       // every branch incl. over/underflow
        if ((i & 15) == 0) {                                                    // raw bit patterns
            double x;
            uint64_t u = rng();
            std::memcpy(&x, &u, 8);
            check(x);
        }
    }
    const double edges[] = {0.0, -0.0, 1e-300, -1e-300, 5e-324, -5e-324, 0x1p-54, -0x1p-54, 0x1p-55, 1.0, -1.0,
                            -708.39, -708.40, -709.0, -744.44, -745.0, -745.13, -745.14, -746.0, 709.78, 709.79,
                            710.0, 1023.9, -1023.9, 1024.0, -1024.0, INFINITY, -INFINITY, NAN};
    for (double x : edges) check(x);
    for (double x = -760.0; x < 720.0; x += 1.0 / 1024) check(x);                // dense grid over the special range
    std::printf("tested %ld arguments, %ld mismatches\n", tested, bad);
    return bad != 0;
}
