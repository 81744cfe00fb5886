// Prints std::to_chars(v) (the reference CLI's fmt_double, proj/tools/chebfilter.cpp:25-29)
// for every bit pattern read from stdin as a 16-digit hex word, one per line.
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
int main() {
    unsigned long long bits;
    while (std::scanf("%llx", &bits) == 1) {
        double v;
        std::memcpy(&v, &bits, 8);
        char b[64];
        auto r = std::to_chars(b, b + sizeof(b), v);
        *r.ptr = 0;
        std::printf("%s\n", b);
    }
}
