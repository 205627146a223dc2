// knobs.cpp -- kernel-variant switches (common.cuh).
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"

namespace ihomgpu {

namespace {
std::mutex g_mu;
std::map<std::string, int>& table() {
  static std::map<std::string, int> t;
  return t;
}
}  // namespace

int knob(const char* name, int dflt) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto& t = table();
  auto it = t.find(name);
  if (it != t.end()) return it->second;
  const std::string env = std::string("IHOM_") + name;
  const char* e = std::getenv(env.c_str());
  const int v = e ? (std::string(e) == "tile" ? 1 : std::atoi(e)) : dflt;
  t.emplace(name, v);
  return v;
}

void set_knob(const char* name, int value) {
  std::lock_guard<std::mutex> lk(g_mu);
  table()[name] = value;
}

}  // namespace ihomgpu
