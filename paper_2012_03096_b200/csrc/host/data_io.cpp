// Dataset producers: the reference's synthetic stripe images and the
// CIFAR-10 binary reader (dataset.cpp:17-134).  The synthetic pixels are
// interface-dictated (bit-exact: the same mt19937_64 streams, distribution
// objects and float arithmetic order as the reference), so their formula is
// the reference's; the rendering loop and the reader are this project's.
#include <algorithm>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <numbers>
#include <random>
#include <thread>

#include "pbkd/dataset.hpp"

namespace pbkd {

namespace {

constexpr int kClasses = 10, kChannels = 3, kSide = 16;
constexpr float kPi = std::numbers::pi_v<float>;

// one image: a sine stripe per class (orientation label%5, frequency 2 or 4),
// per-image phase and amplitude, per-pixel Gaussian noise, clamped to [0,1]
void stripe_image(float* px, int label, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> phase_of(0.0f, 2.0f * kPi);
    std::uniform_real_distribution<float> amp_of(0.7f, 1.0f);
    std::normal_distribution<float> noise(0.0f, 0.05f);
    const float theta = kPi * static_cast<float>(label % 5) / 5.0f;
    const float freq = label < 5 ? 2.0f : 4.0f;
    const float phase = phase_of(rng);  // draw order: phase, amplitude, then pixels
    const float amp = amp_of(rng);
    const float ct = std::cos(theta), st = std::sin(theta);
    const float chan_scale[kChannels] = {1.0f, 0.75f, 0.5f};
    for (int ch = 0; ch < kChannels; ++ch)
        for (int y = 0; y < kSide; ++y) {
            const float v = static_cast<float>(y) / (kSide - 1) - 0.5f;
            for (int x = 0; x < kSide; ++x) {
                const float u = static_cast<float>(x) / (kSide - 1) - 0.5f;
                const float s = std::sin(2.0f * kPi * freq * (ct * u + st * v) + phase);
                *px++ = std::clamp(0.5f + 0.5f * amp * s * chan_scale[ch] + noise(rng), 0.0f, 1.0f);
            }
        }
}

}  // namespace

Dataset make_synthetic_dataset(int count, uint64_t seed, int threads) {
    if (count < 1) throw std::invalid_argument("make_synthetic_dataset: count must be >= 1");
    if (threads < 1) throw std::invalid_argument("make_synthetic_dataset: threads must be >= 1");
    Dataset d;
    d.c = kChannels;
    d.h = d.w = kSide;
    d.classes = kClasses;
    d.labels.resize(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) d.labels[static_cast<size_t>(i)] = i % kClasses;
    d.images.resize(static_cast<size_t>(count) * d.image_size());
    const int workers = std::min(threads, count);
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t)
        pool.emplace_back([&, t] {  // images t, t+workers, ... (independent seeds)
            for (int i = t; i < count; i += workers)
                stripe_image(d.images.data() + static_cast<size_t>(i) * d.image_size(), d.labels[static_cast<size_t>(i)],
                             mix_seed(seed, static_cast<uint64_t>(i)));
        });
    for (std::thread& th : pool) th.join();
    return d;
}

Dataset load_cifar10(const std::string& path) {
    namespace fs = std::filesystem;
    constexpr size_t kPixels = 3 * 32 * 32, kRecord = kPixels + 1;
    std::vector<std::string> files;
    std::error_code ec;
    if (fs::is_directory(path, ec)) {
        for (const auto& e : fs::directory_iterator(path))
            if (e.path().extension() == ".bin") files.push_back(e.path().string());
        std::sort(files.begin(), files.end());
        if (files.empty()) throw std::invalid_argument("load_cifar10: no .bin files in directory " + path);
    } else {
        files.push_back(path);
    }
    Dataset d;
    d.c = 3;
    d.h = d.w = 32;
    d.classes = 10;
    for (const std::string& file : files) {
        std::ifstream in(file, std::ios::binary);
        if (!in) throw std::invalid_argument("load_cifar10: cannot open " + file);
        const std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        if (bytes.empty() || bytes.size() % kRecord != 0)
            throw std::invalid_argument("load_cifar10: " + file + " size " + std::to_string(bytes.size()) +
                                        " is not a multiple of " + std::to_string(kRecord));
        const size_t records = bytes.size() / kRecord;
        d.images.reserve(d.images.size() + records * kPixels);
        for (size_t r = 0; r < records; ++r) {
            const unsigned char* rec = bytes.data() + r * kRecord;
            if (rec[0] > 9)
                throw std::invalid_argument("load_cifar10: " + file + " record " + std::to_string(r) + " has label " +
                                            std::to_string(rec[0]));
            d.labels.push_back(rec[0]);
            for (size_t i = 1; i <= kPixels; ++i) d.images.push_back(static_cast<float>(rec[i]) / 255.0f);
        }
    }
    return d;
}

}  // namespace pbkd
