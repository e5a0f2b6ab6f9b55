// placeholder, replaced by the sfconv:: drop-in
