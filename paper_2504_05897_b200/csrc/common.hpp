// Shared helpers for the C ABI: thread-local error text, status plumbing,
// ExpertRef packing.  No C++ exception ever crosses the extern "C" boundary:
// each entry point wraps its body in HM_API_BEGIN / HM_API_END.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/hybrimoe.h"

namespace hm {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);
const std::string &last_error();

[[noreturn]] inline void raise(int code, const std::string &msg) { throw Error(code, msg); }

inline uint32_t pack_ref(int layer, int expert) {
  return (static_cast<uint32_t>(layer) << 16) | static_cast<uint32_t>(expert);
}
inline int ref_layer(uint32_t r) { return static_cast<int>(r >> 16); }
inline int ref_expert(uint32_t r) { return static_cast<int>(r & 0xffffu); }
inline std::string ref_str(uint32_t r) {
  char b[64];
  std::snprintf(b, sizeof b, "ExpertRef(layer=%d, expert=%d)", ref_layer(r), ref_expert(r));
  return b;
}

}  // namespace hm

#define HM_API_BEGIN try {
#define HM_API_END                                  \
  }                                                 \
  catch (const hm::Error &e) {                      \
    hm::set_last_error(e.what());                   \
    return e.code;                                  \
  }                                                 \
  catch (const std::exception &e) {                 \
    hm::set_last_error(e.what());                   \
    return HM_ERUNTIME;                             \
  }                                                 \
  return HM_OK;

#define HM_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) hm::raise((code), (msg)); \
  } while (0)
