// Runner for the doctest shim -- TEST INFRASTRUCTURE ONLY (see doctest.h).
#include <doctest.h>

#include <cstdio>
#include <cstring>
#include <exception>

int main(int argc, char** argv)
{
    const char* filter = argc > 1 ? argv[1] : nullptr;
    auto& s = doctest::detail::stats();
    int cases = 0;
    for (const auto& tc : doctest::detail::registry()) {
        if (filter && !std::strstr(tc.name, filter))
            continue;
        s.current = tc.name;
        ++cases;
        try {
            tc.fn();
        } catch (const std::exception& e) {
            ++s.failures;
            std::printf("%s:%d: TEST CASE THREW in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
        }
    }
    std::printf("[doctest-shim] test cases: %d | checks: %ld | failed: %ld\n", cases, s.checks, s.failures);
    return s.failures ? 1 : 0;
}
