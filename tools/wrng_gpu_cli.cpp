// wrng-gpu: the reference CLI's subcommands (tools/main.cpp) with the B200
// backend, written against the drop-in header
// wrng_gpu/wallace.hpp — the same calls the reference CLI makes on
// wrng::WallaceState (main.cpp:82-142), so it doubles as a check that an
// existing caller switches by changing one include and one link line.
//
//   gen     finite batch (text | f64le), optional resumable --state-file
//   stream  unbounded raw stream to stdout (SIGPIPE = clean exit)
//   test    statistical suite on the device: uniformity, moments, sumsq
//   bench   throughput: wallace-gpu, boxmuller-gpu, polar-gpu
// Exit codes as main.cpp:27-30: 0 ok/pass, 1 test failure, 2 usage error,
// 3 state-file error.  Flags keep the reference's names and defaults; the
// GPU additions are --n-arrays, --fp32, --pools and --device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <csignal>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "wrng_gpu/wallace.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitTestFail = 1;
constexpr int kExitUsage = 2;
constexpr int kExitStateFile = 3;

struct Options {
    std::string cmd;
    std::uint64_t seed = 1;
    std::uint64_t stream_id = 0;
    std::uint64_t count = 10;
    double mu = 0.0;
    double sigma = 1.0;
    std::uint32_t f = 3;
    std::uint32_t pool_exponent = 10;
    std::string format;  // per-command default
    std::string state_file;
    std::string suite = "all";
    std::vector<std::string> methods = {"wallace-gpu", "polar-gpu", "boxmuller-gpu"};
    double seconds = 1.0;
    std::uint64_t samples = 0;
    // B200 extensions
    std::uint32_t n_arrays = 2;
    bool fp32 = false;
    std::uint32_t pools = 0;  // 0: 1 for gen/stream/test, 8 x SMs for bench
    std::int32_t device = 0;
};

[[noreturn]] void usage(const std::string& why) {
    std::fprintf(stderr,
                 "wrng-gpu: %s\n"
                 "usage: wrng-gpu {gen|stream|test|bench} [--seed S] [--stream-id I] [--f F]\n"
                 "         [--pool-exponent P (8..20)] [--n-arrays 2|4] [--fp32] [--pools K]\n"
                 "         [--device D]\n"
                 "  gen:    [--count C] [--mu M] [--sigma S] [--format text|f64le]\n"
                 "          [--state-file PATH]\n"
                 "  stream: [--mu M] [--sigma S] [--format f64le|text]\n"
                 "  test:   [--suite uniformity|moments|sumsq|all] [--samples N]\n"
                 "  bench:  [--methods wallace-gpu,polar-gpu,boxmuller-gpu] [--seconds T]\n",
                 why.c_str());
    std::exit(kExitUsage);
}

bool parse_u64(const std::string& s, std::uint64_t& out) {
    if (s.empty() || s[0] == '-') return false;
    char* end = nullptr;
    errno = 0;
    const unsigned long long v = std::strtoull(s.c_str(), &end, 0);
    if (errno || *end) return false;
    out = v;
    return true;
}

bool parse_f64(const std::string& s, double& out) {
    char* end = nullptr;
    out = std::strtod(s.c_str(), &end);
    return !s.empty() && !*end && std::isfinite(out);
}

Options parse(int argc, char** argv) {
    Options o;
    if (argc < 2) usage("a subcommand is required");
    o.cmd = argv[1];
    if (o.cmd != "gen" && o.cmd != "stream" && o.cmd != "test" && o.cmd != "bench")
        usage("unknown subcommand '" + o.cmd + "'");
    auto allowed = [&](const std::string& k) {
        static const char* common[] = {"seed", "stream-id", "f", "pool-exponent", "n-arrays",
                                       "fp32", "pools", "device"};
        for (const char* c : common)
            if (k == c) return true;
        if (o.cmd == "gen")
            return k == "count" || k == "mu" || k == "sigma" || k == "format" ||
                   k == "state-file";
        if (o.cmd == "stream") return k == "mu" || k == "sigma" || k == "format";
        if (o.cmd == "test") return k == "suite" || k == "samples";
        return k == "methods" || k == "seconds";
    };
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--", 0) != 0) usage("unexpected argument '" + a + "'");
        std::string key = a.substr(2), val;
        const size_t eq = key.find('=');
        if (eq != std::string::npos) {
            val = key.substr(eq + 1);
            key = key.substr(0, eq);
        } else if (key != "fp32") {
            if (i + 1 >= argc) usage("--" + key + " needs a value");
            val = argv[++i];
        }
        if (!allowed(key)) usage("unknown option --" + key + " for " + o.cmd);
        std::uint64_t u = 0;
        double d = 0;
        if (key == "seed") {
            if (!parse_u64(val, o.seed)) usage("--seed: not an unsigned integer");
        } else if (key == "stream-id") {
            if (!parse_u64(val, o.stream_id)) usage("--stream-id: not an unsigned integer");
        } else if (key == "f") {  // main.cpp:375-376: PositiveNumber
            if (!parse_u64(val, u) || u < 1 || u > 0xFFFFFFFFu) usage("--f must be >= 1");
            o.f = (std::uint32_t)u;
        } else if (key == "pool-exponent") {  // main.cpp:377-379: Range(8, 20)
            if (!parse_u64(val, u) || u < 8 || u > 20) usage("--pool-exponent must be in [8, 20]");
            o.pool_exponent = (std::uint32_t)u;
        } else if (key == "count") {
            if (!parse_u64(val, o.count)) usage("--count: not an unsigned integer");
        } else if (key == "mu") {
            if (!parse_f64(val, o.mu)) usage("--mu: not a number");
        } else if (key == "sigma") {  // NonNegativeNumber
            if (!parse_f64(val, d) || d < 0) usage("--sigma must be >= 0");
            o.sigma = d;
        } else if (key == "format") {
            if (val != "text" && val != "f64le") usage("--format must be text or f64le");
            o.format = val;
        } else if (key == "state-file") {
            o.state_file = val;
        } else if (key == "suite") {
            if (val != "uniformity" && val != "moments" && val != "sumsq" && val != "all" &&
                val != "autocorr")
                usage("--suite must be uniformity, moments, autocorr, sumsq or all");
            o.suite = val;
        } else if (key == "samples") {
            if (!parse_u64(val, o.samples) || o.samples == 0) usage("--samples must be > 0");
        } else if (key == "methods") {
            o.methods.clear();
            size_t p = 0;
            while (p <= val.size()) {
                size_t q = val.find(',', p);
                if (q == std::string::npos) q = val.size();
                std::string m = val.substr(p, q - p);
                // the reference names select the GPU implementations
                if (m == "wallace" || m == "polar" || m == "boxmuller") m += "-gpu";
                if (m != "wallace-gpu" && m != "polar-gpu" && m != "boxmuller-gpu")
                    usage("--methods: unknown method '" + m + "'");
                o.methods.push_back(m);
                p = q + 1;
            }
        } else if (key == "seconds") {
            if (!parse_f64(val, d) || d <= 0) usage("--seconds must be > 0");
            o.seconds = d;
        } else if (key == "n-arrays") {
            if (!parse_u64(val, u) || (u != 2 && u != 4)) usage("--n-arrays must be 2 or 4");
            o.n_arrays = (std::uint32_t)u;
        } else if (key == "fp32") {
            o.fp32 = true;
        } else if (key == "pools") {
            if (!parse_u64(val, u) || u < 1 || u > (1u << 20)) usage("--pools must be >= 1");
            o.pools = (std::uint32_t)u;
        } else if (key == "device") {
            if (!parse_u64(val, u) || u > 63) usage("--device: bad ordinal");
            o.device = (std::int32_t)u;
        }
    }
    if (o.format.empty()) o.format = o.cmd == "stream" ? "f64le" : "text";
    return o;
}

wrng::WallaceConfig make_config(const Options& o, std::uint64_t seed, std::uint32_t pools) {
    wrng::WallaceConfig c;  // main.cpp:48-55
    c.pool_exponent = o.pool_exponent;
    c.throwaway_f = o.f;
    c.seed = seed;
    c.stream_id = o.stream_id;
    c.n_arrays = o.n_arrays;
    c.fp32 = o.fp32;
    c.pools = pools;
    c.device = o.device;
    return c;
}

// Values leave in blocks sized for the GPU path: one device fill and one
// device-to-host copy per 2^20 normals (the stream is the same for any
// blocking, WallaceState::fill continues it).
constexpr size_t kBlockValues = size_t(1) << 20;

// stdout in one of the CLI's two wire formats (proj/tools/main.cpp:59-80
// defines them): "text" — one "%.17g" per line; anything else — raw
// little-endian IEEE-754 doubles.  One byte buffer per block, one fwrite.
class Sink {
public:
    explicit Sink(const std::string& format) : text_(format == "text") {}

    // false once stdout stops taking data (closed pipe, full device)
    bool put(const double* v, size_t n) {
        bytes_.clear();
        if (text_) {
            char line[48];
            for (size_t i = 0; i < n; ++i) {
                const int len = std::snprintf(line, sizeof line, "%.17g\n", v[i]);
                bytes_.insert(bytes_.end(), line, line + len);
            }
        } else {
            bytes_.resize(n * sizeof(double));
            for (size_t i = 0; i < n; ++i) {
                std::uint64_t w;
                std::memcpy(&w, v + i, sizeof w);
                unsigned char* dst = bytes_.data() + i * sizeof w;
                for (unsigned k = 0; k < sizeof w; ++k, w >>= 8) dst[k] = (unsigned char)w;
            }
        }
        return std::fwrite(bytes_.data(), 1, bytes_.size(), stdout) == bytes_.size();
    }
    bool flush() { return std::fflush(stdout) == 0; }

private:
    bool text_;
    std::vector<unsigned char> bytes_;
};

// The generator a command runs on: restored from --state-file when that file
// exists, freshly seeded otherwise.  rc != kExitOk: the file was malformed
// (reported on stderr, exit code of proj/tools/main.cpp:84-100).
std::unique_ptr<wrng::WallaceState> open_generator(const Options& o, int& rc) {
    rc = kExitOk;
    if (!o.state_file.empty()) {
        std::ifstream f(o.state_file, std::ios::binary);
        if (f) {
            const std::vector<std::uint8_t> image{std::istreambuf_iterator<char>(f),
                                                  std::istreambuf_iterator<char>()};
            try {
                return std::make_unique<wrng::WallaceState>(
                    wrng::WallaceState::load_state(image, o.device));
            } catch (const wrng::malformed_state_error& e) {
                std::fprintf(stderr, "wrng-gpu: %s: %s\n", o.state_file.c_str(), e.what());
                rc = kExitStateFile;
                return nullptr;
            }
        }
    }
    return std::make_unique<wrng::WallaceState>(make_config(o, o.seed, o.pools ? o.pools : 1));
}

// Writes the generator's state image back (proj/tools/main.cpp:116-127).
int close_generator(const Options& o, const wrng::WallaceState& st) {
    if (o.state_file.empty()) return kExitOk;
    const auto image = st.save_state();
    std::ofstream f(o.state_file, std::ios::binary | std::ios::trunc);
    f.write(reinterpret_cast<const char*>(image.data()), (std::streamsize)image.size());
    if (f) return kExitOk;
    std::fprintf(stderr, "wrng-gpu: cannot write %s\n", o.state_file.c_str());
    return kExitStateFile;
}

// ---------------------------------------------------------------- gen
int cmd_gen(const Options& o) {
    int rc;
    const auto st = open_generator(o, rc);
    if (!st) return rc;
    Sink sink(o.format);
    std::vector<double> block((size_t)std::min<std::uint64_t>(o.count, kBlockValues));
    for (std::uint64_t sent = 0; sent < o.count;) {
        const size_t n = (size_t)std::min<std::uint64_t>(o.count - sent, block.size());
        st->fill(std::span<double>(block.data(), n), o.mu, o.sigma);
        if (!sink.put(block.data(), n)) break;
        sent += n;
    }
    sink.flush();
    return close_generator(o, *st);
}

// ---------------------------------------------------------------- stream
// Until the consumer closes the pipe, which is a clean exit
// (proj/tools/main.cpp:133-141).
int cmd_stream(const Options& o) {
    std::signal(SIGPIPE, SIG_IGN);
    wrng::WallaceState st(make_config(o, o.seed, o.pools ? o.pools : 1));
    Sink sink(o.format);
    std::vector<double> block(kBlockValues);
    while (true) {
        st.fill(std::span<double>(block), o.mu, o.sigma);
        if (!sink.put(block.data(), block.size()) || !sink.flush()) break;
    }
    return kExitOk;
}

// ---------------------------------------------------------------- test
// One verdict line per check, in the reference CLI's column layout
// (proj/tools/main.cpp:147-158), and the counts the summary needs.
struct Tally {
    int tests = 0, failed = 0;
    void line(const std::string& name, double statistic, const std::string& thr, bool pass) {
        tests += 1;
        if (!pass) failed += 1;
        std::printf("%-34s statistic=%-12.5g threshold=%-22s %s\n", name.c_str(), statistic,
                    thr.c_str(), pass ? "PASS" : "FAIL");
    }
};

void test_uniformity(const Options& o, Tally& t) {
    // main.cpp:160-204 for the Wallace generator: 5 seeds, u and v chi-squared
    // with 1000 bins each, pass band [842, 1156], >= 4 of 5 seeds
    const std::uint64_t pairs = o.samples ? o.samples : 1000000;
    int ok_u = 0, ok_v = 0;
    for (std::uint64_t seed = 1; seed <= 5; ++seed) {
        wrng::WallaceState st(make_config(o, seed, 1));
        const wrng_gpu_validation v = st.validate(2 * pairs, 1000, 1);
        const bool pu = v.u_statistic >= 842.0 && v.u_statistic <= 1156.0;
        const bool pv = v.v_statistic >= 842.0 && v.v_statistic <= 1156.0;
        ok_u += pu;
        ok_v += pv;
        std::printf("uniformity.wallace-gpu.seed%-12llu u=%.1f v=%.1f\n",
                    (unsigned long long)seed, v.u_statistic, v.v_statistic);
    }
    t.line("uniformity.wallace-gpu.u", ok_u, ">=4/5 seeds in [842,1156]", ok_u >= 4);
    t.line("uniformity.wallace-gpu.v", ok_v, ">=4/5 seeds in [842,1156]", ok_v >= 4);
}

void test_moments(const Options& o, Tally& t) {
    // main.cpp:214-230
    const std::uint64_t n = o.samples ? o.samples : 10000000;
    wrng::WallaceState st(make_config(o, o.seed, 1));
    const wrng_gpu_validation v = st.validate(n, 2, 1);
    const double b1 = 4.0 / std::sqrt(double(n));
    const double b2 = 4.0 * std::sqrt(2.0 / double(n));
    const double b4 = 4.0 * std::sqrt(96.0 / double(n));
    char thr[48];
    std::snprintf(thr, sizeof thr, "|m1| <= %.3g", b1);
    t.line("moments.mean", v.m1, thr, std::abs(v.m1) <= b1);
    std::snprintf(thr, sizeof thr, "|m2-1| <= %.3g", b2);
    t.line("moments.second", v.m2, thr, std::abs(v.m2 - 1.0) <= b2);
    std::snprintf(thr, sizeof thr, "|m4-3| <= %.3g", b4);
    t.line("moments.fourth", v.m4, thr, std::abs(v.m4 - 3.0) <= b4);
}

void test_sumsq(const Options& o, Tally& t) {
    // main.cpp:258-268 with sumsq_distribution_check (stats.cpp:129-148)
    if (o.n_arrays != 2) {
        std::printf("sumsq: the suite's target (nu = 2N) is the n = 2 generator's; skipped\n");
        return;
    }
    const std::uint64_t passes = o.samples ? o.samples : 10000;
    wrng::WallaceState st(make_config(o, o.seed, 1));
    double sum = 0.0, sumsq = 0.0;
    for (std::uint64_t i = 0; i < passes; ++i) {
        const double s = st.advance_pass().target_sumsq;
        sum += s;
        sumsq += s * s;
    }
    const double mean = sum / double(passes);
    const double var = sumsq / double(passes) - mean * mean;
    const double nu = 2.0 * double(1u << o.pool_exponent);
    char thr[48];
    std::snprintf(thr, sizeof thr, "within 10%% of %.0f", nu);
    t.line("sumsq.mean", mean, thr, std::abs(mean - nu) <= 0.1 * nu);
    std::snprintf(thr, sizeof thr, "within 30%% of %.0f", 2.0 * nu);
    t.line("sumsq.variance", var, thr, std::abs(var - 2.0 * nu) <= 0.3 * 2.0 * nu);
}

int cmd_test(const Options& o) {
    Tally t;
    if (o.suite == "uniformity" || o.suite == "all") test_uniformity(o, t);
    if (o.suite == "moments" || o.suite == "all") test_moments(o, t);
    if (o.suite == "autocorr")
        std::printf("autocorr: the reference suite runs on its diagnostic pool streams "
                    "(out of scope for the GPU backend); skipped\n");
    if (o.suite == "sumsq" || o.suite == "all") test_sumsq(o, t);
    std::printf("summary tests=%d failed=%d result=%s\n", t.tests, t.failed,
                t.failed == 0 ? "PASS" : "FAIL");
    return t.failed == 0 ? kExitOk : kExitTestFail;
}

// ---------------------------------------------------------------- bench
// main.cpp:287-322 on the device: each method fills a 2^26-value device
// buffer repeatedly (pools = 8 per SM unless --pools) until --seconds pass.
double bench_ns_per_value(const Options& o, const std::string& m, std::uint32_t pools) {
    const size_t block = (size_t)1 << 26;
    const size_t esz = o.fp32 ? 4 : 8;
    void* dev = nullptr;
    if (cudaSetDevice(o.device) != cudaSuccess || cudaMalloc(&dev, block * esz) != cudaSuccess)
        throw wrng::device_error("bench: cannot allocate the device buffer");
    std::unique_ptr<wrng::WallaceState> st;
    if (m == "wallace-gpu") st = std::make_unique<wrng::WallaceState>(make_config(o, o.seed, pools));
    auto one = [&] {
        if (st) {
            if (o.fp32)
                st->fill_device(static_cast<float*>(dev), block, 0.0, 1.0, nullptr);
            else
                st->fill_device(static_cast<double*>(dev), block, 0.0, 1.0, nullptr);
        } else {
            const wrng_gpu_status s = wrng_gpu_method_fill(
                m == "boxmuller-gpu" ? 0 : 1, o.seed, o.stream_id, pools, dev, o.fp32 ? 1 : 0,
                block, 0.0, 1.0, 1, o.device, nullptr);
            if (s != WRNG_GPU_OK) throw wrng::device_error("bench: method fill failed");
        }
    };
    one();  // warm-up
    cudaDeviceSynchronize();
    std::uint64_t produced = 0;
    double elapsed = 0.0;
    const auto start = std::chrono::steady_clock::now();
    do {
        one();
        cudaDeviceSynchronize();
        produced += block;
        elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    } while (elapsed < o.seconds);
    if (st) st->synchronize();
    cudaFree(dev);
    return elapsed * 1e9 / double(produced);
}

int cmd_bench(const Options& o) {
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, o.device);
    const std::uint32_t pools = o.pools ? o.pools : 8u * (std::uint32_t)dev_sms;
    std::printf("%-14s %14s %14s\n", "method", "ns/value", "Mvalues/s");
    for (const std::string& m : o.methods) {
        const double ns = bench_ns_per_value(o, m, pools);
        std::printf("%-14s %14.4f %14.1f\n", m.c_str(), ns, 1000.0 / ns);
        std::printf("bench.%s.ns_per_value=%.5f\n", m.c_str(), ns);
    }
    return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
    const Options o = parse(argc, argv);
    try {
        if (o.cmd == "gen") return cmd_gen(o);
        if (o.cmd == "stream") return cmd_stream(o);
        if (o.cmd == "test") return cmd_test(o);
        return cmd_bench(o);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "wrng-gpu: %s\n", e.what());
        return kExitUsage;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "wrng-gpu: %s\n", e.what());
        return 4;
    }
}
