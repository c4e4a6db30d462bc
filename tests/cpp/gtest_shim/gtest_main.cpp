// gtest_shim runner: runs every registered TEST in registration order, prints
// GoogleTest-style progress, exits nonzero when any test failed. Optional argument
// --gtest_filter=SUBSTR runs only tests whose "Suite.Name" contains SUBSTR.
// Test infrastructure only.
#include <gtest/gtest.h>

namespace gshim {

int run_all(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
    int ran = 0, failed = 0;
    std::vector<std::string> failed_names;
    for (auto& e : registry()) {
        const std::string full = e.suite + "." + e.name;
        if (!filter.empty() && full.find(filter) == std::string::npos) continue;
        ++ran;
        state() = State{};
        testing::UnitTest::GetInstance()->current = {e.suite, e.name};
        std::printf("[ RUN      ] %s\n", full.c_str());
        std::fflush(stdout);
        std::unique_ptr<testing::Test> t;
        try {
            t.reset(e.make());
            t->SetUp();
            if (!state().fatal) t->TestBody();
            t->TearDown();
        } catch (const std::exception& ex) {
            ++state().failures;
            std::fprintf(stderr, "unexpected exception: %s\n", ex.what());
        } catch (...) {
            ++state().failures;
            std::fprintf(stderr, "unexpected exception\n");
        }
        if (state().failures) {
            ++failed;
            failed_names.push_back(full);
            std::printf("[  FAILED  ] %s\n", full.c_str());
        } else {
            std::printf("[       OK ] %s\n", full.c_str());
        }
    }
    std::printf("[==========] %d tests ran.\n[  PASSED  ] %d tests.\n", ran, ran - failed);
    for (auto& n : failed_names) std::printf("[  FAILED  ] %s\n", n.c_str());
    return failed ? 1 : 0;
}

}  // namespace gshim

int main(int argc, char** argv) { return gshim::run_all(argc, argv); }
