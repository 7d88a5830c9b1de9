// dropin_samples.cpp — TEST INFRASTRUCTURE (oracle/Makefile `dropin`): the
// reference's aggregate_samples (samples.cpp:31-85, compiled in place with
// -Daggregate_samples=aggregate_samples_reference) against the libstg C++ shim's
// strata::aggregate_samples (GPU) on
//   * the stream of the reference's own micro-benchmark BM_Aggregation
//     (benchmarks/bench.cpp:79-100: 100k samples, 16 stacks x 12 frames), and
//   * random multi-binary streams with gaps, repeats and several drain intervals.
// Prints one PASS/FAIL line per case and the wall time of both sides.
#include <chrono>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "strata/samples.hpp"

namespace strata {
std::vector<ProfileWindow> aggregate_samples_reference(const std::vector<StackSample>& stream,
                                                       int64_t drain_interval_ns);
}

using namespace strata;

namespace {

bool same(const std::vector<ProfileWindow>& a, const std::vector<ProfileWindow>& b) {
    if (a.size() != b.size()) return false;
    for (size_t w = 0; w < a.size(); ++w) {
        if (a[w].rank != b[w].rank || a[w].window_start_ns != b[w].window_start_ns ||
            a[w].window_end_ns != b[w].window_end_ns || a[w].records.size() != b[w].records.size())
            return false;
        for (size_t r = 0; r < a[w].records.size(); ++r)
            if (a[w].records[r].count != b[w].records[r].count || !(a[w].records[r].frames == b[w].records[r].frames))
                return false;
    }
    return true;
}

std::vector<StackSample> bench_stream() {  // bench.cpp:80-95
    BuildId id = BuildId::digest(std::string_view("a"));
    std::mt19937_64 rng(7);
    std::vector<std::vector<FrameRef>> pool;
    for (int s = 0; s < 16; ++s) {
        std::vector<FrameRef> stack;
        for (int d = 0; d < 12; ++d) stack.push_back({id, 0x1000 + uint64_t(s * 64 + d * 8)});
        pool.push_back(std::move(stack));
    }
    std::vector<StackSample> stream;
    std::uniform_int_distribution<size_t> pick(0, pool.size() - 1);
    for (int i = 0; i < 100'000; ++i) {
        StackSample s;
        s.timestamp_ns = int64_t(i) * 10'000;
        s.frames = pool[pick(rng)];
        stream.push_back(std::move(s));
    }
    return stream;
}

std::vector<StackSample> random_stream(uint64_t seed, int n, int64_t t0) {
    std::mt19937_64 rng(seed);
    std::vector<BuildId> ids;
    for (int b = 0; b < 3; ++b) ids.push_back(BuildId::digest("bin" + std::to_string(b)));
    std::vector<std::vector<FrameRef>> pool;
    for (int s = 0; s < 200; ++s) {
        std::vector<FrameRef> st;
        int d = 1 + int(rng() % 30);
        for (int k = 0; k < d; ++k) st.push_back({ids[rng() % 3], 0x400 + (rng() % 512) * 4});
        pool.push_back(st);
        if (s % 5 == 0) {  // near duplicates: other binary on the root frame, one frame shorter
            auto v = st;
            v.back().build_id = ids[(rng() % 2 + 1 + 0) % 3];
            pool.push_back(v);
            if (st.size() > 1) pool.push_back(std::vector<FrameRef>(st.begin(), st.end() - 1));
        }
    }
    std::vector<StackSample> out(n);
    int64_t t = t0;
    for (int i = 0; i < n; ++i) {
        uint64_t r = rng() % 1000;
        t += r < 100 ? 0 : (r < 998 ? int64_t(rng() % 20'000'000) : 9'000'000'000);
        out[i].timestamp_ns = t;
        out[i].rank = 5;
        out[i].frames = pool[std::min<size_t>(pool.size() - 1, size_t(rng() % pool.size()) * (rng() % 3 == 0 ? 0 : 1))];
    }
    return out;
}

double secs(std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

}  // namespace

int main() {
    int fails = 0;
    auto run = [&](const char* name, const std::vector<StackSample>& s, int64_t drain) {
        auto t0 = std::chrono::steady_clock::now();
        auto ref = aggregate_samples_reference(s, drain);
        double tr = secs(t0);
        aggregate_samples(s, drain);  // warm (context, staging)
        t0 = std::chrono::steady_clock::now();
        auto got = aggregate_samples(s, drain);
        double tg = secs(t0);
        bool ok = same(ref, got);
        fails += !ok;
        std::printf("%s %s: %zu samples, %zu windows; reference %.2f ms, libstg %.2f ms\n", ok ? "PASS" : "FAIL",
                    name, s.size(), ref.size(), tr * 1e3, tg * 1e3);
    };
    run("bench.cpp BM_Aggregation stream", bench_stream(), 5'000'000'000);
    run("random stream, 5 s drain", random_stream(1, 200'000, 3'000'000'000), 5'000'000'000);
    run("random stream, 1 ms drain", random_stream(2, 200'000, -77'000'000), 1'000'000);
    run("random stream, 1 ns drain", random_stream(3, 50'000, 0), 1);
    // errors must carry the reference's messages
    auto expect_throw = [&](const char* name, const std::vector<StackSample>& s, int64_t drain) {
        std::string a = "-", b = "-";
        try { aggregate_samples_reference(s, drain); } catch (const Error& e) { a = e.what(); }
        try { aggregate_samples(s, drain); } catch (const Error& e) { b = e.what(); }
        bool ok = a == b && a != "-";
        fails += !ok;
        std::printf("%s %s: \"%s\"\n", ok ? "PASS" : "FAIL", name, b.c_str());
    };
    auto bad = random_stream(4, 1000, 0);
    bad[500].frames.clear();
    expect_throw("empty stack", bad, 5'000'000'000);
    bad = random_stream(5, 1000, 0);
    bad[300].timestamp_ns -= 1'000'000'000;
    expect_throw("regression", bad, 5'000'000'000);
    bad = random_stream(6, 1000, 0);
    bad[700].rank = 6;
    expect_throw("mixed ranks", bad, 5'000'000'000);
    expect_throw("drain", random_stream(7, 10, 0), 0);
    std::printf("%s\n", fails ? "FAILED" : "ALL PASS");
    return fails ? 1 : 0;
}
