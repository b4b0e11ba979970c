// ctx.hpp -- the C ABI context (include/pbkd_b200.h pbkd_ctx), shared by the
// ABI translation units.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "../comm.hpp"
#include "../engine.hpp"

struct pbkd_ctx {
    // the context's GPUs: eng on devices[0], peers on devices[1..]
    std::unique_ptr<pbkd_gpu::Engine> eng;
    std::vector<std::unique_ptr<pbkd_gpu::Engine>> peers;
    // created over a device list (pbkd_ctx_create_multi): the engines share
    // one in-process NCCL clique and run_parallel spreads its workers over
    // them (runtime.cpp:226-233, a host thread per GPU)
    bool multi = false;
    std::string spec;
    std::vector<pbkd_gpu::Engine*> engines() const {
        std::vector<pbkd_gpu::Engine*> v{eng.get()};
        for (const auto& p : peers) v.push_back(p.get());
        return v;
    }
};
