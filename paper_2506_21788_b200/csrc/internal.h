// internal.h -- declarations shared by host.cpp, ctx.cu and comm.cpp.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "hmtl_b200.h"

namespace hmtl_b200 {

struct LayoutEntry {
  std::string name;
  size_t rows, cols, offset;
};
struct Layout {
  std::vector<LayoutEntry> entries;
  size_t total = 0;
  const LayoutEntry& at(const std::string& n) const {
    for (const auto& e : entries)
      if (e.name == n) return e;
    return entries.front();
  }
};

Layout make_layout(const hmtl_hyper& hp, bool shared);
void init_block(const hmtl_hyper& hp, uint64_t seed, int which, float* out);
uint64_t seed_stream(uint64_t master, uint64_t id);
int fail(int code, const std::string& msg);
int hmtp_write(const char* path, const hmtl_hyper& hp, const float* shared, size_t ps, const float* const* heads,
               size_t ph, int n_heads, const hmtl_ckpt_opt* opt);
int hmtp_read(const char* path, hmtl_hyper* hp, std::vector<double>* shared, std::vector<std::vector<double>>* heads,
              bool* has_opt, uint64_t* step, std::vector<std::vector<double>>* opt_blocks);
extern thread_local std::string g_last_error;

}  // namespace hmtl_b200
